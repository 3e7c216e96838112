// K2f (segmented fill) — the fill pass of the owned-mask build (conflict.py:119-161: the
// re-scan that writes every admitted partner, then the canonical CSR with rows ascending).
//
// One warp per row, per-warp bitmap over an id window [w0, w0 + wb).  Three phases per window:
//
//  1. decode: the row's owned mask rows (one per color, conflict-pair ownership makes them
//     disjoint) are cut into 32-position words.  A word is decoded by the whole warp: lane t
//     loads bucket member 32w+t (one coalesced 128-byte load) and the mask word (one broadcast
//     load); an admitted member sets its bit with a plain shared load/or/store, verified, and
//     re-applied with an atomic only when another lane of the same instruction hit the same
//     word (rare: members of one bucket are ~n/m ids apart).  The words of every color are
//     flattened into a descriptor list first, so loads of 8 words are in flight per lane.
//  2. count: lane l owns bitmap words [l*S, l*S+S) — a contiguous id segment — and popcounts
//     them; a warp exclusive scan gives every lane the output position of its segment.
//     S is odd, so the loads of the 32 lanes hit 32 distinct banks.
//     The count pass also records the lane's nonzero words (a 64-bit summary; S <= 63).
//  3. extract: each lane visits only its nonzero words (ascending), clears them and emits
//     their ids (three unrolled, a rarely taken loop for more) into its own contiguous run of
//     the row's output slice.  Sparse rows (1M ids, ~3k entries) skip the empty words.
//
// Windows: n <= wb is one window (config 2: 100k ids = 12.8 KB of bitmap).  Larger n uses
// per-color window bounds (k_window_bounds: members below each window start), and a word that
// straddles two windows is decoded in both, filtered by id range.
#include <algorithm>
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

constexpr int SEG_MAX_WARPS = 4;
constexpr int SEG_CH = 8;  // descriptor words decoded per step

__device__ __forceinline__ uint32_t s_lds(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void s_sts(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 s_lds4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void s_sts4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint32_t s_lds_if(bool p, uint32_t addr) {
    uint32_t v = 0u;
    asm volatile(
        "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
        : "+r"(v)
        : "r"(addr), "r"((uint32_t)p)
        : "memory");
    return v;
}
__device__ __forceinline__ void s_sts_if(bool p, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}

__device__ __forceinline__ int seg_excl_scan(int v, int lane, int &total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

// Per-lane color slot: bucket start in bmemp, first mask word of the row's owned mask row,
// words of the mask row (W), bucket size (m), color.
struct Slot {
    int32_t b = 0, W = 0, c = 0;
    uint32_t r = 0;
};

__device__ __forceinline__ Slot load_slot(const RowArgs &a, int64_t lo, int Li, int s) {
    Slot sl;
    if (s < Li) {
        const int c = a.lrel[lo + s];
        const int m = a.bstart[c + 1] - a.bstart[c];
        sl.c = c;
        sl.W = (m + 31) >> 5;
        sl.b = a.bpos[c];
        sl.r = (uint32_t)(a.maskoff[c] + (int64_t)a.posof[lo + s] * sl.W);
    }
    return sl;
}

__device__ __forceinline__ uint32_t s_lds16(uint32_t addr) {
    unsigned short v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void s_sts16(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}

template <typename OutT, bool MULTI, bool COMPACT>
__global__ void __launch_bounds__(SEG_MAX_WARPS * 32) k_fill_seg(RowArgs a, SegArgs g) {
    extern __shared__ __align__(16) uint32_t ssm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwarps = blockDim.x >> 5;
    const int WW = g.wb >> 5;   // bitmap words = 32 * S
    const int S = g.seg;        // words per lane segment (odd)
    // per warp: bitmap (WW words) | 32 dummy words | descriptors
    uint32_t *bm = ssm + (size_t)warp * g.warp_words;
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(bm);
    const uint32_t dummy_s = bm_s + (uint32_t)(WW + lane) * 4u;
    int2 *desc = reinterpret_cast<int2 *>(bm + WW + 32);
    const uint32_t seg_s = bm_s + (uint32_t)(lane * S) * 4u;
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    __syncwarp();

    OutT *out = reinterpret_cast<OutT *>(a.out);
    // opaque per-lane base pointer: keeps each gather at one IMAD.WIDE.U32
    const int32_t *bmem_l;
    asm("mov.b64 %0, %1;" : "=l"(bmem_l) : "l"(a.bmemp + lane));
    const uint32_t *masks = a.masks;
    const int32_t *compact = a.compact;
    const uint32_t lanebit = 1u << lane;
    const int64_t stride = (int64_t)gridDim.x * nwarps;
    for (int64_t ri = a.row_begin + (int64_t)blockIdx.x * nwarps + warp; ri < a.row_end;
         ri += stride) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        if (a.deg[i] == 0) continue;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        const Slot s0 = load_slot(a, lo, Li, lane);
        const Slot s1 = load_slot(a, lo, Li, lane + 32);
        OutT *orow = out + (a.rowoff[i] - a.out_base);
        for (int k = 0; k < g.nwin; ++k) {
            const int32_t w0 = k * g.wb;
            const uint32_t wlen = (uint32_t)(min((int64_t)a.n, (int64_t)w0 + g.wb) - w0);
            const uint32_t wbase_s = bm_s - (uint32_t)(w0 >> 5) * 4u;  // bitmap word of id 0
            // ---- descriptors of the words of this window, flattened over the row's colors:
            // (first bucket position of the word, the owned mask word itself)
            int lo0 = 0, n0 = s0.W, lo1 = 0, n1 = s1.W;
            if (MULTI) {
                const int st = g.nwin + 1;
                if (lane < Li) {
                    const int p0 = g.bnd[(int64_t)s0.c * st + k], p1 = g.bnd[(int64_t)s0.c * st + k + 1];
                    lo0 = p0 >> 5;
                    n0 = p1 > p0 ? ((p1 + 31) >> 5) - lo0 : 0;
                }
                if (lane + 32 < Li) {
                    const int p0 = g.bnd[(int64_t)s1.c * st + k], p1 = g.bnd[(int64_t)s1.c * st + k + 1];
                    lo1 = p0 >> 5;
                    n1 = p1 > p0 ? ((p1 + 31) >> 5) - lo1 : 0;
                }
            }
            int T0, T1;
            const int off0 = seg_excl_scan(n0, lane, T0);
            const int off1 = seg_excl_scan(n1, lane, T1);
#pragma unroll 4
            for (int q = 0; q < n0; ++q)
                desc[off0 + q] = make_int2(s0.b + 32 * (lo0 + q), (int)__ldg(masks + s0.r + (uint32_t)(lo0 + q)));
            for (int q = 0; q < n1; ++q)
                desc[T0 + off1 + q] = make_int2(s1.b + 32 * (lo1 + q), (int)__ldg(masks + s1.r + (uint32_t)(lo1 + q)));
            const int T = T0 + T1;
            const int T8 = (T + SEG_CH - 1) & ~(SEG_CH - 1);  // padded: unpredicated loads
            if (T + lane < T8) desc[T + lane] = make_int2(0, 0);  // (mask 0: nothing admitted)
            __syncwarp();
            // ---- decode: mark admitted ids in the bitmap (plain load/or/store; non-admitted
            // lanes touch their own dummy word: no predicates to keep alive across phases)
            for (int f0 = 0; f0 < T8; f0 += SEG_CH) {
                uint32_t addr[SEG_CH], bit[SEG_CH];
#pragma unroll
                for (int u = 0; u < SEG_CH; ++u) {
                    const int2 d = desc[f0 + u];
                    const int32_t x = __ldg(bmem_l + (uint32_t)d.x);
                    bool adm = ((uint32_t)d.y & lanebit) != 0u;
                    if (MULTI) adm = adm && (uint32_t)(x - w0) < wlen;
                    // w0 is a multiple of 32: the window base folds into the bitmap address
                    addr[u] = adm ? wbase_s + ((uint32_t)x >> 5) * 4u : dummy_s;
                    bit[u] = adm ? (1u << (x & 31)) : 0u;
                }
                uint32_t old[SEG_CH];
#pragma unroll
                for (int u = 0; u < SEG_CH; ++u) old[u] = s_lds(addr[u]);
#pragma unroll
                for (int u = 0; u < SEG_CH; ++u) s_sts(addr[u], old[u] | bit[u]);
                __syncwarp();
                uint32_t lost = 0u;
#pragma unroll
                for (int u = 0; u < SEG_CH; ++u) {
                    old[u] = bit[u] & ~s_lds(addr[u]);  // bits lost to a same-word store
                    lost |= old[u];
                }
                if (__any_sync(0xffffffffu, lost != 0u)) {
#pragma unroll
                    for (int u = 0; u < SEG_CH; ++u)
                        if (old[u]) atomicOr(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(addr[u])), old[u]);
                }
                __syncwarp();
            }
            // ---- count: lane l owns words [l*S, l*S+S) — a contiguous id segment (S odd: the
            // 32 lanes' loads hit 32 distinct banks).  The same pass records which of the
            // lane's words are nonzero (S <= 63 bits), so extraction touches only those.
            int cnt = 0;
            uint32_t ra = 0u, rb = 0u;  // nonzero flags, shifted in (word q at bit S1-1-q)
            const int S1 = min(S, 32);
#pragma unroll 4
            for (int q = 0; q < S1; ++q) {
                const uint32_t v = s_lds(seg_s + (uint32_t)q * 4u);
                cnt += __popc(v);
                ra = (ra << 1) | min(v, 1u);
            }
#pragma unroll 4
            for (int q = 32; q < S; ++q) {
                const uint32_t v = s_lds(seg_s + (uint32_t)q * 4u);
                cnt += __popc(v);
                rb = (rb << 1) | min(v, 1u);
            }
            uint32_t nz0 = __brev(ra) >> (32 - S1);                  // bit q <-> word q
            uint32_t nz1 = S > 32 ? __brev(rb) >> (64 - S) : 0u;     // bit q-32 <-> word q
            int tot;
            const int pos = seg_excl_scan(cnt, lane, tot);
            // ---- extract: each step takes the lane's next nonzero word, clears it and emits
            // its ids (three unrolled; a rarely taken loop for more) into the lane's own run of
            // the row's output slice
            OutT *op = orow + pos;
            const int32_t cb0 = (MULTI ? w0 : 0) + lane * S * 32;
            uint64_t nz = ((uint64_t)nz1 << 32) | nz0;
            int e = 0;
            while (__any_sync(0xffffffffu, nz != 0ull)) {
                if (nz == 0ull) continue;
                const int q = __ffsll((long long)nz) - 1;
                nz &= nz - 1ull;
                uint32_t v = s_lds(seg_s + (uint32_t)q * 4u);
                s_sts(seg_s + (uint32_t)q * 4u, 0u);
                const int32_t cb = cb0 + q * 32;
                {
                    const int32_t j = cb + __ffs(v) - 1;
                    v &= v - 1u;
                    op[e++] = (OutT)(COMPACT ? __ldg(compact + j) : j);
                }
                if (v) {
                    const int32_t j = cb + __ffs(v) - 1;
                    v &= v - 1u;
                    op[e++] = (OutT)(COMPACT ? __ldg(compact + j) : j);
                }
                if (v) {
                    const int32_t j = cb + __ffs(v) - 1;
                    v &= v - 1u;
                    op[e++] = (OutT)(COMPACT ? __ldg(compact + j) : j);
                }
                while (v) {  // words with 4+ ids
                    const int32_t j = cb + __ffs(v) - 1;
                    v &= v - 1u;
                    op[e++] = (OutT)(COMPACT ? __ldg(compact + j) : j);
                }
            }
            orow += tot;
            __syncwarp();
        }
    }
}

// bnd[c * (nwin + 1) + k] = members of bucket c with id < k * wb (bucket members ascend).
__global__ void k_window_bounds(const int32_t *__restrict__ bstart, const int32_t *__restrict__ bpos,
                                const int32_t *__restrict__ bmemp, int64_t P, int nwin, int32_t wb,
                                int32_t *__restrict__ bnd) {
    const int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int st = nwin + 1;
    if (x >= P * st) return;
    const int64_t c = x / st;
    const int k = (int)(x % st);
    const int m = bstart[c + 1] - bstart[c];
    const int32_t *mem = bmemp + bpos[c];
    const int64_t lim = (int64_t)k * wb;
    int lo = 0, hi = m;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if ((int64_t)mem[mid] < lim) lo = mid + 1; else hi = mid;
    }
    bnd[x] = lo;
}

template <typename OutT, bool MULTI, bool COMPACT>
int run_seg(const RowArgs &a, const SegArgs &g, int sms, cudaStream_t s) {
    const int warps = std::max(1, std::min(SEG_MAX_WARPS, g.warps));
    const size_t smem = (size_t)g.warp_words * 4 * warps;
    auto kern = k_fill_seg<OutT, MULTI, COMPACT>;
    allow_max_smem(kern);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, warps * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)per_sm * sms, (rows + warps - 1) / warps));
    kern<<<(unsigned)grid, warps * 32, smem, s>>>(a, g);
    return 1;
}

}  // namespace

// Window geometry: words per lane S (multiple of 4, S/4 odd: conflict-free 128-bit segment
// loads), window wb = 1024*S bits.  `max_bits` caps the per-warp bitmap.
void seg_geometry(int64_t n, int64_t max_bits, int32_t *wb, int32_t *nwin, int32_t *seg) {
    // S words per lane, S odd (conflict-free lane-segment loads); the window is 1024*S ids
    int64_t smax = std::min<int64_t>(63, std::max<int64_t>(1, max_bits / 1024));
    if ((smax & 1) == 0) smax -= 1;
    int64_t S = (std::max<int64_t>(n, 1) + 1023) / 1024;
    if ((S & 1) == 0) S += 1;
    if (S > smax) S = smax;
    *seg = (int32_t)S;
    *wb = (int32_t)(1024 * S);
    *nwin = (int32_t)((std::max<int64_t>(n, 1) + *wb - 1) / *wb);
}

int launch_window_bounds(const int32_t *bstart, const int32_t *bpos, const int32_t *bmemp,
                         int64_t P, int nwin, int32_t wb, int32_t *bnd, cudaStream_t s) {
    const int64_t total = P * (nwin + 1);
    if (total == 0) return 0;
    k_window_bounds<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(bstart, bpos, bmemp, P, nwin,
                                                                    wb, bnd);
    return 1;
}

int launch_fill_seg(const RowArgs &a, const SegArgs &g, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    const bool c = a.compact != nullptr;
    if (g.nwin > 1) {
        if (c) return out64 ? run_seg<int64_t, true, true>(a, g, sms, s) : run_seg<int32_t, true, true>(a, g, sms, s);
        return out64 ? run_seg<int64_t, true, false>(a, g, sms, s) : run_seg<int32_t, true, false>(a, g, sms, s);
    }
    if (c) return out64 ? run_seg<int64_t, false, true>(a, g, sms, s) : run_seg<int32_t, false, true>(a, g, sms, s);
    return out64 ? run_seg<int64_t, false, false>(a, g, sms, s) : run_seg<int32_t, false, false>(a, g, sms, s);
}

}  // namespace pcg
