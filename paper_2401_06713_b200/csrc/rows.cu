// K2 — conflict rows.  For every row i of the build, the admitted partners
//     { j != i : list(i) ∩ list(j) != ∅  and  parity(popc(A_i & B_j)) == 0 }
// (conflict.py:72-78: edge & (mask_i & mask_j).any()), produced in ascending j, i.e.
// directly in the canonical CSR row order of conflict.py:148-161 — no sort pass.
//
// Exact list intersection without the reference's dense ceil(P/64)-word masks: the
// candidates of row i are the union of its L color buckets (bucket c = ascending local ids
// holding color c).  Two variants, bit-identical results:
//
//  * bucket-mask mode (default):
//      K2a (color-major) k_bucket_masks — for every color c with members v_0 < ... < v_{m-1},
//          the m x m commute matrix mask_c[k][t] = commute(v_k, v_t) && k != t, as m rows of
//          ceil(m/32) words.  A member's partner vector is loaded once per color (one
//          broadcast per warp) instead of once per (row, candidate): sum_c m_c = n*L loads
//          instead of sum_c m_c^2 gathers.
//      K2b (row-major) k_rows_masked — row i is member k of bucket c in each of its L
//          colors; its admitted partners through c are the set bits of mask_c[k], in member
//          order.  No partner vectors are touched.
//  * gather mode (k_rows; dense corners where the masks would not fit): every candidate's
//    partner vector is gathered and the predicate evaluated in the row pass.
//
// Both row passes: one warp per row, the id range swept in windows of `window` ids; lane s
// walks bucket s of the row (8 members per round, all loads in flight) and admitted members
// set their bit in a per-warp shared-memory bitmap of the window, which deduplicates
// partners shared through several colors and sorts them.  Marking is a plain load / or /
// store per round plus one verify pass; only bits lost to a same-word store of the same round
// are re-applied with an atomic (shared atomics cost ~2 cycles per lane, so they stay off the
// common path).  Harvest: lane l owns a contiguous segment of the window; the count pass
// popcounts it (degree, and upper degree j > i), the fill pass takes a warp exclusive scan of
// the segment popcounts and writes ids in ascending order.  Rows are independent: the
// multi-GPU path gives each GPU a row range.
#include <algorithm>
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

constexpr int RW_WARPS = 8;
constexpr int UNR = 8;          // bucket members per lane per round
constexpr int MASK_KG = 4;      // rows of one color per lane per pass in K2a (32*KG per pass)
constexpr int MASK_WARPS = 8;
constexpr int STAGE = 1024;     // fill-pass staging (ids per warp)

template <int KW>
struct RowVec {
    uint32_t v[KW > 0 ? KW : 1];
    __device__ __forceinline__ void load(const uint32_t *A, int64_t i, int kw) {
#pragma unroll
        for (int k = 0; k < KW; ++k) v[k] = __ldg(A + i * KW + k);
    }
    __device__ __forceinline__ uint32_t parity(const uint32_t *B, int32_t j, int kw) const {
        uint32_t acc = 0;
        const uint32_t *b = B + (int64_t)j * KW;
        if constexpr (KW % 4 == 0) {
#pragma unroll
            for (int k = 0; k < KW; k += 4) {
                const uint4 w = __ldg(reinterpret_cast<const uint4 *>(b + k));
                acc ^= (v[k] & w.x) ^ (v[k + 1] & w.y) ^ (v[k + 2] & w.z) ^ (v[k + 3] & w.w);
            }
        } else if constexpr (KW % 2 == 0) {
#pragma unroll
            for (int k = 0; k < KW; k += 2) {
                const uint2 w = __ldg(reinterpret_cast<const uint2 *>(b + k));
                acc ^= (v[k] & w.x) ^ (v[k + 1] & w.y);
            }
        } else {
#pragma unroll
            for (int k = 0; k < KW; ++k) acc ^= v[k] & __ldg(b + k);
        }
        return __popc(acc) & 1u;
    }
};

// Runtime-width fallback (very long strings / raw mode with odd widths).
template <>
struct RowVec<0> {
    const uint32_t *a;
    __device__ __forceinline__ void load(const uint32_t *A, int64_t i, int kw) { a = A + i * kw; }
    __device__ __forceinline__ uint32_t parity(const uint32_t *B, int32_t j, int kw) const {
        uint32_t acc = 0;
        const uint32_t *b = B + (int64_t)j * kw;
        for (int k = 0; k < kw; ++k) acc ^= __ldg(a + k) & __ldg(b + k);
        return __popc(acc) & 1u;
    }
};

__device__ __forceinline__ int warp_excl_scan(int v, int lane, int &total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 lds_u128(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void sts_u128(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// Popcount of the bits of one 128-bit harvest chunk (ids jlo .. jlo+127) above `self`.
__device__ __forceinline__ int upper_count(uint4 q, int32_t jlo, int32_t self) {
    if (jlo > self) return __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
    if (jlo + 128 <= self) return 0;
    const uint32_t w[4] = {q.x, q.y, q.z, q.w};
    int c = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int32_t d = self - (jlo + 32 * u);
        const uint32_t m = d < 0 ? 0xffffffffu : (d >= 31 ? 0u : ~((2u << d) - 1u));
        c += __popc(w[u] & m);
    }
    return c;
}

__device__ __forceinline__ uint32_t lds_u32_if(bool p, uint32_t addr) {
    uint32_t v = 0u;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "r"(addr), "r"((uint32_t)p)
        : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32_if(bool p, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}

// Marks up to UNR admitted bits per lane (bit == 0: nothing to mark; those accesses are
// predicated off so they cost no shared-memory wavefronts).  Plain load / or / store, then
// one verify; bits lost to a same-word store of this round go through an atomic.
__device__ __forceinline__ void mark_round(const uint32_t (&addr)[UNR], const uint32_t (&bit)[UNR]) {
    uint32_t old[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) old[u] = lds_u32_if(bit[u] != 0u, addr[u]);
#pragma unroll
    for (int u = 0; u < UNR; ++u) sts_u32_if(bit[u] != 0u, addr[u], old[u] | bit[u]);
    __syncwarp();
    uint32_t lost = 0u;
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
        old[u] = bit[u] & ~lds_u32_if(bit[u] != 0u, addr[u]);
        lost |= old[u];
    }
    if (__any_sync(0xffffffffu, lost != 0u)) {
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            if (old[u])
                atomicOr(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(addr[u])), old[u]);
    }
    __syncwarp();
}

// Harvest of one window.  Chunks are interleaved across lanes (lane l reads 16-byte chunk
// it*32 + l), so every LDS.128 / STS.128 is conflict-free; ids keep ascending order because
// chunk index grows with (it, lane).  Count pass: degree and upper degree.  Fill pass: per
// chunk row a warp exclusive scan orders the ids; they are extracted into the warp's shared
// staging buffer and stored to global memory coalesced.  Clears the bitmap.
template <bool FILL, typename OutT>
__device__ __forceinline__ void harvest(uint32_t bm_s, int WW, int32_t w0, int32_t self, int lane,
                                        int &cnt, int &cntu, int64_t &outpos, OutT *out,
                                        const int32_t *compact, int32_t *stage) {
    const int rows = WW >> 7;  // 128 words (32 lanes x 4) per chunk row
    if constexpr (!FILL) {
        for (int it = 0; it < rows; ++it) {
            const int c = it * 32 + lane;
            const uint32_t addr = bm_s + (uint32_t)c * 16u;
            const uint4 q4 = lds_u128(addr);
            if ((q4.x | q4.y | q4.z | q4.w) == 0u) continue;
            sts_u128(addr, make_uint4(0u, 0u, 0u, 0u));
            cnt += __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
            cntu += upper_count(q4, w0 + c * 128, self);
        }
    } else {
        int fillv = 0;  // ids currently staged
        for (int it = 0; it < rows; ++it) {
            const int c = it * 32 + lane;
            const uint32_t addr = bm_s + (uint32_t)c * 16u;
            const uint4 q4 = lds_u128(addr);
            const int nb = __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
            int total;
            const int base = warp_excl_scan(nb, lane, total);
            if (total == 0) continue;
            const bool direct = total > STAGE;  // dense chunk row: store straight out
            if (fillv > 0 && (direct || fillv + total > STAGE)) {
                __syncwarp();
                for (int k = lane; k < fillv; k += 32) out[outpos + k] = (OutT)stage[k];
                outpos += fillv;
                fillv = 0;
                __syncwarp();
            }
            if (nb) {
                sts_u128(addr, make_uint4(0u, 0u, 0u, 0u));
                int64_t pos = direct ? outpos + base : fillv + base;
                const uint32_t wv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t wd = wv[u];
                    const int32_t jb = w0 + c * 128 + 32 * u;
                    while (wd) {
                        const int b = __ffs(wd) - 1;
                        wd &= wd - 1u;
                        const int32_t j = jb + b;
                        const int32_t val = compact ? compact[j] : j;
                        if (direct) out[pos++] = (OutT)val;
                        else stage[pos++] = val;
                    }
                }
            }
            if (direct) {
                outpos += total;  // staging was flushed before this row
            } else {
                fillv += total;
            }
        }
        __syncwarp();
        for (int k = lane; k < fillv; k += 32) out[outpos + k] = (OutT)stage[k];
        outpos += fillv;
        __syncwarp();
    }
}

template <bool FILL>
__device__ __forceinline__ void finish_row(int64_t i, int lane, int cnt, int cntu, int32_t *deg,
                                           int32_t *degu) {
    if constexpr (!FILL) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_down_sync(0xffffffffu, cnt, o);
            cntu += __shfl_down_sync(0xffffffffu, cntu, o);
        }
        if (lane == 0) {
            deg[i] = cnt;
            degu[i] = cntu;
        }
    }
}

// ---------------------------------------------------------------------------------------
// gather mode
// ---------------------------------------------------------------------------------------
template <int KW, bool FILL, typename OutT>
__global__ void __launch_bounds__(RW_WARPS * 32) k_rows(RowArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int WW = a.window >> 5;
    const int slots = (2 * a.slot_cap + 3) & ~3;
    uint32_t *bm = smem + (size_t)warp * (WW + 32 + STAGE + slots);
    int32_t *stage = reinterpret_cast<int32_t *>(bm + WW + 32);
    int32_t *cur = stage + STAGE;
    int32_t *cend = cur + a.slot_cap;
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(bm);
    const uint32_t dummy_s = bm_s + (uint32_t)(WW + lane) * 4u;
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    __syncwarp();

    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int64_t stride = (int64_t)gridDim.x * RW_WARPS;
    for (int64_t ri = a.row_begin + (int64_t)blockIdx.x * RW_WARPS + warp; ri < a.row_end;
         ri += stride) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        for (int s = lane; s < Li; s += 32) {
            const int c = a.lrel[lo + s];
            cur[s] = a.bstart[c];
            cend[s] = a.bstart[c + 1];
        }
        RowVec<KW> ai;
        ai.load(a.A, i, a.kw);
        __syncwarp();
        int cnt = 0, cntu = 0;
        int64_t outpos = FILL ? (a.rowoff[i] - a.out_base) : 0;
        const int32_t self = (int32_t)i;
        for (int32_t w0 = 0; w0 < a.n; w0 += a.window) {
            const int32_t w1 = (int32_t)min((int64_t)a.n, (int64_t)w0 + a.window);
            for (int sg = 0; sg < Li; sg += 32) {
                const int s = sg + lane;
                const bool act = s < Li;
                int p = act ? cur[s] : 0;
                const int e = act ? cend[s] : 0;
                bool go = act && p < e;
                while (__any_sync(0xffffffffu, go)) {
                    int m[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u)
                        m[u] = (go && p + u < e) ? __ldg(a.bmem + p + u) : INT_MAX;
                    int k = 0;
#pragma unroll
                    for (int u = 0; u < UNR; ++u) k += m[u] < w1 ? 1 : 0;
                    p += k;
                    go = go && k == UNR;
                    uint32_t addr[UNR], bit[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const bool adm = m[u] < w1 && m[u] != self &&
                                         ai.parity(a.B, m[u], a.kw) == 0u;
                        const uint32_t off = (uint32_t)(m[u] - w0);
                        addr[u] = adm ? bm_s + ((off >> 5) << 2) : dummy_s;
                        bit[u] = adm ? (1u << (off & 31)) : 0u;
                    }
                    mark_round(addr, bit);
                }
                if (act) cur[s] = p;
            }
            __syncwarp();
            harvest<FILL, OutT>(bm_s, WW, w0, self, lane, cnt, cntu, outpos, out, a.compact, stage);
            __syncwarp();
        }
        finish_row<FILL>(i, lane, cnt, cntu, a.deg, a.degu);
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// bucket-mask mode: K2a
// ---------------------------------------------------------------------------------------
__global__ void k_bucket_layout(BucketArgs b, int64_t entries) {
    const int64_t pos = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (pos >= entries) return;
    const int32_t e = b.sorted_e[pos];
    int64_t lo = 0, hi = b.P;  // color of this sorted position (bstart is monotone)
    while (hi - lo > 1) {
        const int64_t mid = (lo + hi) >> 1;
        if (b.bstart[mid] <= pos) lo = mid; else hi = mid;
    }
    const int32_t t = (int32_t)(pos - b.bstart[lo]);
    const int32_t r = b.row_of[e];
    b.bmemp[b.bpos[lo] + t] = r;
    b.posof[e] = t;
    if (b.bmem) b.bmem[pos] = r;
}

template <int KW>
__global__ void __launch_bounds__(MASK_WARPS * 32) k_bucket_masks(BucketArgs b) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)MASK_WARPS + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * MASK_WARPS;
    for (int64_t c = gw; c < b.P; c += nw) {
        const int m = b.bstart[c + 1] - b.bstart[c];
        if (m < 2) {
            if (m == 1 && lane == 0) b.masks[b.maskoff[c]] = 0u;
            continue;
        }
        const int W = (m + 31) >> 5;
        const int32_t *mem = b.bmemp + b.bpos[c];
        uint32_t *out = b.masks + b.maskoff[c];
        for (int kb = 0; kb < m; kb += 32 * MASK_KG) {
            RowVec<KW> ak[MASK_KG];
            int kk[MASK_KG];
#pragma unroll
            for (int g = 0; g < MASK_KG; ++g) {
                kk[g] = kb + 32 * g + lane;
                ak[g].load(b.A, kk[g] < m ? mem[kk[g]] : mem[0], b.kw);
            }
            for (int w = 0; w < W; ++w) {
                uint32_t bits[MASK_KG];
#pragma unroll
                for (int g = 0; g < MASK_KG; ++g) bits[g] = 0u;
                const int tend = min(32, m - 32 * w);
                for (int tt = 0; tt < tend; ++tt) {
                    const int t = 32 * w + tt;
                    const int32_t j = mem[t];  // same address in every lane: one broadcast
#pragma unroll
                    for (int g = 0; g < MASK_KG; ++g) {
                        const uint32_t par = ak[g].parity(b.B, j, b.kw);
                        bits[g] |= ((par ^ 1u) & (t != kk[g] ? 1u : 0u)) << tt;
                    }
                }
#pragma unroll
                for (int g = 0; g < MASK_KG; ++g)
                    if (kk[g] < m) out[(int64_t)kk[g] * W + w] = bits[g];
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// bucket-mask mode: K2b
// ---------------------------------------------------------------------------------------
template <bool FILL, typename OutT>
__global__ void __launch_bounds__(RW_WARPS * 32) k_rows_masked(RowArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int WW = a.window >> 5;
    // per-warp region: bitmap (WW) | 32 dummy words | slot arrays (t, m, base | row int64)
    const int off_r = (3 * a.slot_cap + 1) & ~1;
    const int slot_words = (off_r + 2 * a.slot_cap + 3) & ~3;
    uint32_t *bm = smem + (size_t)warp * (WW + 32 + STAGE + slot_words);
    int32_t *stage = reinterpret_cast<int32_t *>(bm + WW + 32);
    int32_t *st = stage + STAGE;
    int32_t *sm = st + a.slot_cap;
    int32_t *sb = sm + a.slot_cap;
    int64_t *sr = reinterpret_cast<int64_t *>(st + off_r);
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(bm);
    const uint32_t dummy_s = bm_s + (uint32_t)(WW + lane) * 4u;
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    __syncwarp();

    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int64_t stride = (int64_t)gridDim.x * RW_WARPS;
    for (int64_t ri = a.row_begin + (int64_t)blockIdx.x * RW_WARPS + warp; ri < a.row_end;
         ri += stride) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        for (int s = lane; s < Li; s += 32) {
            const int c = a.lrel[lo + s];
            const int m = a.bstart[c + 1] - a.bstart[c];
            st[s] = 0;
            sm[s] = m;
            sb[s] = a.bpos[c];
            sr[s] = a.maskoff[c] + (int64_t)a.posof[lo + s] * ((m + 31) >> 5);
        }
        __syncwarp();
        int cnt = 0, cntu = 0;
        int64_t outpos = FILL ? (a.rowoff[i] - a.out_base) : 0;
        const int32_t self = (int32_t)i;
        for (int32_t w0 = 0; w0 < a.n; w0 += a.window) {
            const int32_t w1 = (int32_t)min((int64_t)a.n, (int64_t)w0 + a.window);
            for (int sg = 0; sg < Li; sg += 32) {
                const int s = sg + lane;
                const bool act = s < Li;
                int t = act ? st[s] : 0;
                const int m = act ? sm[s] : 0;
                const int32_t *mem = a.bmemp + (act ? sb[s] : 0);
                const uint32_t *mrow = a.masks + (act ? sr[s] : 0);
                bool go = act && t < m;
                while (__any_sync(0xffffffffu, go)) {
                    // 8 positions of an 8-aligned group (bucket starts are 4-aligned, padded)
                    const int gs = t & ~(UNR - 1);
                    int4 v0 = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX), v1 = v0;
                    uint32_t mb = 0u;
                    if (go) {
                        v0 = __ldg(reinterpret_cast<const int4 *>(mem + gs));
                        v1 = __ldg(reinterpret_cast<const int4 *>(mem + gs + 4));
                        mb = __ldg(mrow + (gs >> 5)) >> (gs & 31);
                    }
                    const int v[UNR] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
                    uint32_t addr[UNR], bit[UNR];
                    int k = 0;
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        const bool in = (gs + u >= t) & (gs + u < m) & (v[u] < w1);
                        k += in ? 1 : 0;
                        const bool adm = in & ((mb >> u) & 1u);
                        const uint32_t off = (uint32_t)(v[u] - w0);
                        addr[u] = adm ? bm_s + ((off >> 5) << 2) : dummy_s;
                        bit[u] = adm ? (1u << (off & 31)) : 0u;
                    }
                    t += k;
                    go = go && t == gs + UNR && t < m;
                    mark_round(addr, bit);
                }
                if (act) st[s] = t;
            }
            __syncwarp();
            harvest<FILL, OutT>(bm_s, WW, w0, self, lane, cnt, cntu, outpos, out, a.compact, stage);
            __syncwarp();
        }
        finish_row<FILL>(i, lane, cnt, cntu, a.deg, a.degu);
        __syncwarp();
    }
}

size_t gather_warp_bytes(const RowArgs &a) {
    return (size_t)((a.window >> 5) + 32 + STAGE + ((2 * a.slot_cap + 3) & ~3)) * 4;
}
size_t masked_warp_bytes(const RowArgs &a) {
    const int off_r = (3 * a.slot_cap + 1) & ~1;
    return (size_t)((a.window >> 5) + 32 + STAGE + ((off_r + 2 * a.slot_cap + 3) & ~3)) * 4;
}

template <typename Kern>
int launch_row_kernel(Kern k, const RowArgs &a, size_t per_warp, int sms, cudaStream_t s) {
    const size_t smem = per_warp * RW_WARPS;
    allow_max_smem(k);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, RW_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    int64_t grid = (int64_t)per_sm * sms;
    const int64_t need = (rows + RW_WARPS - 1) / RW_WARPS;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    k<<<(unsigned)grid, RW_WARPS * 32, smem, s>>>(a);
    return 1;
}

template <bool FILL, typename OutT>
int dispatch_gather(const RowArgs &a, int sms, cudaStream_t s) {
    const size_t pw = gather_warp_bytes(a);
    switch (a.kw) {
        case 2: return launch_row_kernel(k_rows<2, FILL, OutT>, a, pw, sms, s);
        case 4: return launch_row_kernel(k_rows<4, FILL, OutT>, a, pw, sms, s);
        case 6: return launch_row_kernel(k_rows<6, FILL, OutT>, a, pw, sms, s);
        case 8: return launch_row_kernel(k_rows<8, FILL, OutT>, a, pw, sms, s);
        case 12: return launch_row_kernel(k_rows<12, FILL, OutT>, a, pw, sms, s);
        default: return launch_row_kernel(k_rows<0, FILL, OutT>, a, pw, sms, s);
    }
}

template <bool FILL, typename OutT>
int dispatch_rows(const RowArgs &a, int sms, cudaStream_t s) {
    if (a.masks) return launch_row_kernel(k_rows_masked<FILL, OutT>, a, masked_warp_bytes(a), sms, s);
    return dispatch_gather<FILL, OutT>(a, sms, s);
}

template <int KW>
int run_masks(const BucketArgs &b, int sms, cudaStream_t s) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bucket_masks<KW>, MASK_WARPS * 32, 0);
    if (per_sm < 1) per_sm = 1;
    int64_t grid = (int64_t)per_sm * sms;
    const int64_t need = (b.P + MASK_WARPS - 1) / MASK_WARPS;
    if (grid > need) grid = need;
    k_bucket_masks<KW><<<(unsigned)std::max<int64_t>(grid, 1), MASK_WARPS * 32, 0, s>>>(b);
    return 1;
}

__global__ void k_compact(const int32_t *__restrict__ deg, int64_t n,
                          const int32_t *__restrict__ compact, const int64_t *__restrict__ rowoff,
                          const int64_t *__restrict__ active, int64_t *__restrict__ members,
                          int64_t *__restrict__ offsets, int32_t *__restrict__ mrow) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = deg[i];
    const int64_t k = compact ? compact[i] : i;
    if (d > 0) {
        members[k] = active[i];
        offsets[k] = rowoff[i];
        if (mrow) mrow[k] = (int32_t)i;  // member -> active row (pipelined public fill)
    }
    if (i == n - 1) offsets[k + (d > 0 ? 1 : 0)] = rowoff[n];
}

}  // namespace

int launch_rows(const RowArgs &a, bool fill, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    if (!fill) return dispatch_rows<false, int32_t>(a, sms, s);
    if (out64) return dispatch_rows<true, int64_t>(a, sms, s);
    return dispatch_rows<true, int32_t>(a, sms, s);
}

int launch_bucket_layout(const BucketArgs &b, int64_t entries, cudaStream_t s) {
    if (entries == 0) return 0;
    const int tb = 256;
    k_bucket_layout<<<(unsigned)((entries + tb - 1) / tb), tb, 0, s>>>(b, entries);
    return 1;
}

int launch_bucket_masks(const BucketArgs &b, int sms, cudaStream_t s) {
    switch (b.kw) {
        case 2: return run_masks<2>(b, sms, s);
        case 4: return run_masks<4>(b, sms, s);
        case 6: return run_masks<6>(b, sms, s);
        case 8: return run_masks<8>(b, sms, s);
        case 12: return run_masks<12>(b, sms, s);
        default: return run_masks<0>(b, sms, s);
    }
}

int launch_compact(const int32_t *deg, int64_t n, const int32_t *compact, const int64_t *rowoff,
                   const int64_t *active, int64_t *members_out, int64_t *offsets_out,
                   int32_t *mrow, cudaStream_t s) {
    if (n == 0) return 0;
    const int tb = 256;
    k_compact<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(deg, n, compact, rowoff, active,
                                                           members_out, offsets_out, mrow);
    return 1;
}

}  // namespace pcg
