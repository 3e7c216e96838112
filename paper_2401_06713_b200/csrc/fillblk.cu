// K2f (block fill) — the fill pass of the owned-mask build (conflict.py:119-161: the re-scan
// that writes every admitted partner, then the canonical CSR with rows ascending), one CTA
// per row over a bitmap of the whole id range (or of wide windows of it).
//
// Per row (per window):
//  A. slots: thread s takes color s of the row's list — its bucket, the row's owned mask row
//     (disjoint across colors by ownership), the mask words that fall in the window — and a
//     block scan flattens the (color, word) pairs into a descriptor list.
//  B. mark: descriptors are materialised in shared memory (thread per descriptor: one mask
//     word load each, all in flight), then each warp decodes 8 at a time: lane t loads bucket
//     member 32w+t (one coalesced 128-byte load) and, if its mask bit is set, ORs its bit into
//     the bitmap (red.shared.or, no return value) and appends the id to the row's list (the
//     mask word is the ballot; one shared reservation per warp batch).
//  C. prefix: the bitmap is cut into 128-id groups (4 words); thread t owns G consecutive
//     groups, popcounts them and a block scan gives every thread its base; each group keeps
//     a 4-byte record: its position relative to the thread's base (11 bits) and the set bits
//     of its first three words (7 bits each, cumulative).  Groups are XOR-swizzled inside
//     each thread's run so the 128-bit loads of a quarter warp hit distinct banks.
//  D. place: every listed id's output index is its thread base + its group's record + the
//     set bits below it in its word, so each entry is written straight to its place in the
//     row (ascending ids), with no per-lane extraction loop.  A window whose ids overflow the
//     list decodes its descriptors again instead.
//  E. clear the bitmap.
// Rows wider than the window (n > NT*G*128 ids) are cut into windows; a mask word straddling
// two windows is decoded in both and filtered by id range (per-color window bounds as in the
// segmented fill).
#include <algorithm>
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

__device__ __forceinline__ uint4 blk_lds4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
// predicated shared/global accesses: the decode loops stay branch-free
__device__ __forceinline__ void blk_red_or_if(bool p, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ void blk_sts_if(bool p, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.u32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ void blk_red_add_if(bool p, uint32_t addr, uint32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q red.shared.add.u32 [%0], %1;\n\t}" ::"r"(addr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ uint32_t blk_lds_if(bool p, uint32_t addr) {
    uint32_t v = 0u;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.u32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "r"(addr), "r"((uint32_t)p)
                 : "memory");
    return v;
}
__device__ __forceinline__ uint2 blk_lds2_if(bool p, uint32_t addr) {
    uint2 v = make_uint2(0u, 0u);
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %3, 0;\n\t@q ld.shared.v2.u32 {%0,%1}, [%2];\n\t}"
                 : "+r"(v.x), "+r"(v.y)
                 : "r"(addr), "r"((uint32_t)p)
                 : "memory");
    return v;
}
__device__ __forceinline__ int32_t blk_ldg_if(bool p, const int32_t *ptr) {
    int32_t v = 0;
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.nc.s32 %0, [%1];\n\t}"
                 : "+r"(v)
                 : "l"(ptr), "r"((uint32_t)p));
    return v;
}
__device__ __forceinline__ void blk_stg_if(bool p, int32_t *ptr, int32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.s32 [%0], %1;\n\t}" ::"l"(ptr),
                 "r"(v), "r"((uint32_t)p)
                 : "memory");
}
__device__ __forceinline__ void blk_stg_if(bool p, int64_t *ptr, int32_t v) {
    asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.global.s64 [%0], %1;\n\t}" ::"l"(ptr),
                 "l"((int64_t)v), "r"((uint32_t)p)
                 : "memory");
}

// block-wide exclusive scan of one int per thread (every thread calls it)
__device__ __forceinline__ int blk_scan(int v, int *wt, int &total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    const int w = lane < nw ? wt[lane] : 0;
    int z = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
    }
    total = __shfl_sync(0xffffffffu, z, 31);
    const int base = __shfl_sync(0xffffffffu, z - w, warp);
    __syncthreads();  // wt is reused by the next scan
    return base + x - v;
}

// physical group of logical group g (thread t = g / G owns G consecutive groups): XOR of the
// low log2(G) bits so that the j-th loads of 8 consecutive threads fall in distinct banks
template <int G>
__device__ __forceinline__ uint32_t blk_swz(uint32_t g) {
    constexpr int LG = G >= 16 ? 4 : G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0;
    if (G == 1) return g;
    const uint32_t t = g >> LG;
    const uint32_t f = G >= 8 ? (t & 7u) : ((t >> (3 - LG)) & (uint32_t)(G - 1));
    return g ^ f;
}

struct BlkLayout {
    uint32_t *bm;     // nga*4 words (bitmap, swizzled groups)
    uint32_t *gp;     // nga, same swizzle: output position of the group relative to its
                      // thread's base (bits 21..31) | set bits in the group's words before
                      // word 1, 2, 3 (7 bits each, cumulative)
    int32_t *tbase;   // threads: output position of each thread's first group
    int32_t *list;    // ecap: the row's admitted ids in this window (any order)
    int2 *desc;       // dcap descriptors: (bucket position of the word, mask word)
    int32_t *sB;      // lcap: bucket position of the slot's first word in the window
    uint32_t *sR;     // lcap: mask word index of the slot's first word in the window
    int32_t *sC;      // lcap: exclusive prefix of the slots' word counts
    int32_t *wt;      // 32: scan scratch
};

// descriptors [cb, cb+nd) of the row's flattened (slot, word) list, padded with empty words
__device__ __forceinline__ void blk_build_desc(const BlkLayout &L, const uint32_t *masks, int cb,
                                               int nd, int T, int Li, uint64_t pol) {
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        const int dd = cb + d;
        int2 v = make_int2(0, 0);
        if (dd < T) {
            int lo_s = 0, hi_s = Li - 1;  // last slot with sC <= dd
            while (lo_s < hi_s) {
                const int mid = (lo_s + hi_s + 1) >> 1;
                if (L.sC[mid] <= dd) lo_s = mid; else hi_s = mid - 1;
            }
            const int q = dd - L.sC[lo_s];
            v = make_int2(L.sB[lo_s] + 32 * q, (int)ldg_pol(masks + L.sR[lo_s] + (uint32_t)q, pol));
        }
        L.desc[d] = v;
    }
}

// output index (within the window's run of the row) of window-relative id xr
template <int G>
__device__ __forceinline__ uint32_t blk_rank(const BlkLayout &L, uint32_t xr) {
    constexpr int LG = G >= 16 ? 4 : G >= 8 ? 3 : G >= 4 ? 2 : G >= 2 ? 1 : 0;
    const uint32_t wi = xr >> 5, lg = wi >> 2, kq = wi & 3u;
    const uint32_t pg = blk_swz<G>(lg);
    const uint32_t e = L.gp[pg];
    const uint32_t wd = L.bm[pg * 4u + kq];
    const uint32_t before = kq ? (e >> (7u * (kq - 1u))) & 127u : 0u;
    return (uint32_t)L.tbase[lg >> LG] + (e >> 21) + before + __popc(wd & ((1u << (xr & 31)) - 1u));
}

template <typename OutT, int G, bool MULTI, bool COMPACT>
__global__ void __launch_bounds__(1024) k_fill_blk(RowArgs a, BlkArgs g) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int NT = blockDim.x, NW = NT >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nga = g.nga;  // bitmap groups (multiple of G)
    BlkLayout L;
    L.bm = sm;
    L.gp = L.bm + (size_t)nga * 4;
    L.tbase = reinterpret_cast<int32_t *>(L.gp + ((nga + 1) & ~1));  // (8-byte alignment below)
    L.list = L.tbase + ((NT + 1) & ~1);
    L.desc = reinterpret_cast<int2 *>(L.list + ((g.ecap + 1) & ~1));
    L.sB = reinterpret_cast<int32_t *>(L.desc + g.dcap);
    L.sR = reinterpret_cast<uint32_t *>(L.sB + g.lcap);
    L.sC = reinterpret_cast<int32_t *>(L.sR + g.lcap);
    L.wt = L.sC + g.lcap;
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(L.bm);
    const uint32_t gp_s = (uint32_t)__cvta_generic_to_shared(L.gp);
    const uint32_t cnt_s = (uint32_t)__cvta_generic_to_shared(L.wt + 32);  // list length
    uint4 *bm4 = reinterpret_cast<uint4 *>(L.bm);
    for (int k = tid; k < nga; k += NT) bm4[k] = make_uint4(0u, 0u, 0u, 0u);

    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int32_t *bmem_l;
    asm("mov.b64 %0, %1;" : "=l"(bmem_l) : "l"(a.bmemp + lane));
    const uint32_t *masks = a.masks;
    const int32_t *compact = a.compact;
    const uint64_t pol_masks = l2_policy_stream();
    const uint32_t lt = (1u << lane) - 1u;
    const bool own_groups = tid * G < nga;  // this thread's groups exist
    __syncthreads();

    for (int64_t ri = a.row_begin + blockIdx.x; ri < a.row_end; ri += gridDim.x) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        if (a.deg[i] == 0) continue;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        OutT *orow = out + (a.rowoff[i] - a.out_base);
        for (int k = 0; k < g.nwin; ++k) {
            const int32_t w0 = MULTI ? k * g.wb : 0;
            const uint32_t wlen = (uint32_t)(min((int64_t)a.n, (int64_t)w0 + g.wb) - w0);
            // ---- A: slots (the row's colors) and their words in this window
            int T = 0;
            for (int s0 = 0; s0 < Li; s0 += NT) {
                const int s = s0 + tid;
                int nw = 0;
                if (s < Li) {
                    const int c = a.lrel[lo + s];
                    const int m = a.bstart[c + 1] - a.bstart[c];
                    const int W = (m + 31) >> 5;
                    int wlo = 0;
                    nw = W;
                    if (MULTI) {
                        const int st = g.nwin + 1;
                        const int p0 = g.bnd[(int64_t)c * st + k], p1 = g.bnd[(int64_t)c * st + k + 1];
                        wlo = p0 >> 5;
                        nw = p1 > p0 ? ((p1 + 31) >> 5) - wlo : 0;
                    }
                    L.sB[s] = a.bpos[c] + 32 * wlo;
                    L.sR[s] = (uint32_t)(a.maskoff[c] + (int64_t)a.posof[lo + s] * W) + (uint32_t)wlo;
                }
                int tot;
                const int ex = blk_scan(nw, L.wt, tot);
                if (s < Li) L.sC[s] = T + ex;
                T += tot;
            }
            if (tid == 0) L.wt[32] = 0;
            __syncthreads();
            if (T == 0) continue;  // uniform: nothing of this row in the window
            const int Tp = (T + 7) & ~7;
            const bool once = Tp <= g.dcap;  // descriptors built once, reused by pass D
            // ---- B: mark (and collect the admitted ids in the row's list while they fit)
            for (int cb = 0; cb < Tp; cb += g.dcap) {
                const int nd = min(Tp - cb, g.dcap);
                blk_build_desc(L, masks, cb, nd, T, Li, pol_masks);
                __syncthreads();
                for (int d0 = warp * 8; d0 < nd; d0 += NW * 8) {
                    int32_t x[8];
                    uint32_t mw[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int2 dv = L.desc[d0 + u];
                        x[u] = __ldg(bmem_l + (uint32_t)dv.x);
                        mw[u] = (uint32_t)dv.y;
                    }
                    uint32_t bal[8];
                    int cnt = 0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        bool adm = ((mw[u] >> lane) & 1u) != 0u;
                        const uint32_t xr = (uint32_t)(x[u] - w0);
                        if (MULTI) adm = adm && xr < wlen;
                        const uint32_t wi = xr >> 5;
                        const uint32_t pg = blk_swz<G>(wi >> 2);
                        blk_red_or_if(adm, bm_s + (pg * 4u + (wi & 3u)) * 4u, 1u << (x[u] & 31));
                        bal[u] = MULTI ? __ballot_sync(0xffffffffu, adm) : mw[u];
                        cnt += __popc(bal[u]);
                    }
                    if (g.ecap > 0) {  // one shared reservation per warp batch (lane 0)
                        uint32_t off = 0;
                        if (lane == 0 && cnt > 0)
                            asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(off) : "r"(cnt_s), "r"(cnt) : "memory");
                        off = __shfl_sync(0xffffffffu, off, 0);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint32_t e = off + __popc(bal[u] & lt);
                            if (((bal[u] >> lane) & 1u) && e < (uint32_t)g.ecap) L.list[e] = x[u];
                            off += __popc(bal[u]);
                        }
                    }
                }
                __syncthreads();
            }
            // ---- C: group positions (thread t: logical groups t*G .. t*G+G-1)
            uint32_t loc[G], cum[G];
            int run = 0;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                uint4 v = make_uint4(0u, 0u, 0u, 0u);
                if (own_groups) v = blk_lds4(bm_s + blk_swz<G>((uint32_t)(tid * G + j)) * 16u);
                const uint32_t c0 = __popc(v.x), c1 = c0 + __popc(v.y), c2 = c1 + __popc(v.z);
                loc[j] = (uint32_t)run;
                cum[j] = c0 | (c1 << 7) | (c2 << 14);
                run += (int)(c2 + __popc(v.w));
            }
            int wtot;
            const int ne = L.wt[32];  // (read before the scan reuses the scratch words)
            const int base = blk_scan(run, L.wt, wtot);
            L.tbase[tid] = base;
            if (own_groups) {
#pragma unroll
                for (int j = 0; j < G; ++j)
                    L.gp[blk_swz<G>((uint32_t)(tid * G + j))] = (loc[j] << 21) | cum[j];
            }
            __syncthreads();
            // ---- D: place every admitted member at its output index
            if (g.ecap > 0 && ne <= g.ecap) {  // from the list: every lane holds an entry
                for (int e0 = tid; e0 < ne; e0 += 4 * NT) {
                    int32_t x[4];
                    uint32_t r[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const int e = e0 + u * NT;
                        x[u] = e < ne ? L.list[e] : w0;
                        r[u] = blk_rank<G>(L, (uint32_t)(x[u] - w0));
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (e0 + u * NT < ne) orow[r[u]] = (OutT)(COMPACT ? __ldg(compact + x[u]) : x[u]);
                }
            } else {  // list overflow: decode the descriptors again
                for (int cb = 0; cb < Tp; cb += g.dcap) {
                    const int nd = min(Tp - cb, g.dcap);
                    if (!once) {
                        blk_build_desc(L, masks, cb, nd, T, Li, pol_masks);
                        __syncthreads();
                    }
                    for (int d0 = warp * 8; d0 < nd; d0 += NW * 8) {
                        int32_t x[8];
                        uint32_t mw[8];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const int2 dv = L.desc[d0 + u];
                            x[u] = __ldg(bmem_l + (uint32_t)dv.x);
                            mw[u] = (uint32_t)dv.y;
                        }
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            bool adm = ((mw[u] >> lane) & 1u) != 0u;
                            const uint32_t xr = (uint32_t)(x[u] - w0);
                            if (MULTI) adm = adm && xr < wlen;
                            uint32_t r = 0;
                            if (adm) r = blk_rank<G>(L, xr);
                            if (adm) orow[r] = (OutT)(COMPACT ? __ldg(compact + x[u]) : x[u]);
                        }
                    }
                    if (!once) __syncthreads();
                }
            }
            __syncthreads();
            // ---- E: clear the bitmap for the next row / window
            for (int q = tid; q < nga; q += NT) bm4[q] = make_uint4(0u, 0u, 0u, 0u);
            orow += wtot;
            // (the next row's slot pass ends with a barrier before anything reads the bitmap)
        }
    }
}

template <typename OutT, int G, bool MULTI, bool COMPACT>
int run_blk(const RowArgs &a, const BlkArgs &g, int sms, cudaStream_t s) {
    const size_t smem = blk_smem_bytes(g, G);
    auto kern = k_fill_blk<OutT, G, MULTI, COMPACT>;
    allow_max_smem(kern);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, g.threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms, rows));
    kern<<<(unsigned)grid, g.threads, smem, s>>>(a, g);
    return 1;
}

template <typename OutT, int G>
int run_blk_g(const RowArgs &a, const BlkArgs &g, int sms, cudaStream_t s) {
    const bool c = a.compact != nullptr;
    if (g.nwin > 1)
        return c ? run_blk<OutT, G, true, true>(a, g, sms, s) : run_blk<OutT, G, true, false>(a, g, sms, s);
    return c ? run_blk<OutT, G, false, true>(a, g, sms, s) : run_blk<OutT, G, false, false>(a, g, sms, s);
}

template <typename OutT>
int run_blk_t(const RowArgs &a, const BlkArgs &g, int sms, cudaStream_t s) {
    switch (g.groups) {
        case 1: return run_blk_g<OutT, 1>(a, g, sms, s);
        case 2: return run_blk_g<OutT, 2>(a, g, sms, s);
        case 4: return run_blk_g<OutT, 4>(a, g, sms, s);
        case 8: return run_blk_g<OutT, 8>(a, g, sms, s);
        default: return run_blk_g<OutT, 16>(a, g, sms, s);
    }
}

// ---------------------------------------------------------------------------------------
// K2f for sparse rows (bins fill): one CTA per row, counting sort instead of a bitmap.  The
// admitted ids of the row are collected in a list while 2^s-id bins count them (s chosen so
// that a bin holds ~1 entry); a block scan turns the counts into bin offsets, the ids are
// scattered into bin order, and an id's output index is its bin's offset + the ids of its
// bin below it (a few comparisons).  No window and no pass over the id range: the work is
// per admitted id and per bin (~n/deg bins), which wins where a row holds a tiny fraction of
// the ids (1M ids, ~3k entries per row).  Used only when the longest row fits the list.
// ---------------------------------------------------------------------------------------
// the k (<= N) ids at src, sorted ascending, to dst[0..k): a bitonic network over N registers
// (padded with INT_MAX), fully unrolled (compile-time indices)
template <int N, typename OutT, bool COMPACT>
__device__ __forceinline__ void bins_sort_out(const int32_t *src, int k, OutT *dst,
                                              const int32_t *compact, uint64_t pol) {
    int32_t v[N];
#pragma unroll
    for (int t = 0; t < N; ++t) v[t] = t < k ? src[t] : INT_MAX;
#pragma unroll
    for (int kk = 2; kk <= N; kk <<= 1) {
#pragma unroll
        for (int j = kk >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const int32_t lo = min(v[i], v[l]), hi = max(v[i], v[l]);
                    if ((i & kk) == 0) { v[i] = lo; v[l] = hi; } else { v[i] = hi; v[l] = lo; }
                }
            }
        }
    }
#pragma unroll
    for (int t = 0; t < N; ++t)
        if (t < k) stg_pol(dst + t, COMPACT ? __ldg(compact + v[t]) : v[t], pol);
}

// 56 registers: six 192-thread CTAs per SM at config 3 (57 would leave five; the shared
// memory also allows six) — the fill is latency-bound and barrier-heavy, more resident rows
// hide both (measured 19.5 -> 17.8 ms at config 3)
template <typename OutT, bool COMPACT>
__global__ void __maxnreg__(56) k_fill_bins(RowArgs a, BinArgs g) {
    extern __shared__ __align__(16) uint32_t sm[];
    const int NT = blockDim.x, NW = NT >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    int32_t *list = reinterpret_cast<int32_t *>(sm);   // ecap: admitted ids, any order
    int32_t *buf = list + g.ecap;                      // ecap: ids in bin order
    int32_t *bins = buf + g.ecap;                      // nbins: counts -> ends of the bins
    BlkLayout L;
    L.desc = reinterpret_cast<int2 *>(bins + ((g.nbins + 1) & ~1));
    L.sB = reinterpret_cast<int32_t *>(L.desc + g.dcap);
    L.sR = reinterpret_cast<uint32_t *>(L.sB + g.lcap);
    L.sC = reinterpret_cast<int32_t *>(L.sR + g.lcap);
    L.wt = L.sC + g.lcap;
    int *count = L.wt + 32;
    for (int b = tid; b < g.nbins; b += NT) bins[b] = 0;

    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int32_t *bmem_l;
    asm("mov.b64 %0, %1;" : "=l"(bmem_l) : "l"(a.bmemp + lane));
    const uint32_t *masks = a.masks;
    const int32_t *compact = a.compact;
    const uint32_t lt = (1u << lane) - 1u;
    const int sh = g.shift;
    const int per = (g.nbins + NT - 1) / NT;  // bins per thread in the scan
    const uint64_t pol_keep = l2_policy_keep(), pol_out = l2_policy_stream(), pol_masks = pol_out;
    const uint32_t list_s = (uint32_t)__cvta_generic_to_shared(list);
    const uint32_t bins_s = (uint32_t)__cvta_generic_to_shared(bins);
    __syncthreads();

    __shared__ long long witem;
    for (int64_t ri = a.row_begin + work_first(a.work, &witem); ri < a.row_end;
         ri = a.row_begin + work_next(a.work, &witem, ri - a.row_begin)) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        if (a.deg[i] == 0) continue;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        OutT *orow = out + (a.rowoff[i] - a.out_base);
        // ---- slots (the row's colors): bucket, owned mask row, words
        int T = 0;
        for (int s0 = 0; s0 < Li; s0 += NT) {
            const int s = s0 + tid;
            int nw = 0;
            if (s < Li) {
                const int c = a.lrel[lo + s];
                const int m = a.bstart[c + 1] - a.bstart[c];
                const int W = (m + 31) >> 5;
                nw = W;
                L.sB[s] = a.bpos[c];
                L.sR[s] = (uint32_t)(a.maskoff[c] + (int64_t)a.posof[lo + s] * W);
            }
            int tot;
            const int ex = blk_scan(nw, L.wt, tot);
            if (s < Li) L.sC[s] = T + ex;
            T += tot;
        }
        if (tid == 0) *count = 0;
        __syncthreads();
        const int Tp = (T + 7) & ~7;
        // ---- collect the admitted ids and count them per bin
        for (int cb = 0; cb < Tp; cb += g.dcap) {
            const int nd = min(Tp - cb, g.dcap);
            blk_build_desc(L, masks, cb, nd, T, Li, pol_masks);
            __syncthreads();
            for (int d0 = warp * 8; d0 < nd; d0 += NW * 8) {
                int32_t x[8];
                uint32_t mw[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int2 dv = L.desc[d0 + u];
                    x[u] = ldg_pol(bmem_l + (uint32_t)dv.x, pol_keep);
                    mw[u] = (uint32_t)dv.y;
                }
                int cnt = 0;
#pragma unroll
                for (int u = 0; u < 8; ++u) cnt += __popc(mw[u]);
                int off = 0;
                if (lane == 0 && cnt > 0) {
                    asm volatile("atom.shared.add.u32 %0, [%1], %2;"
                                 : "=r"(off)
                                 : "r"((uint32_t)__cvta_generic_to_shared(count)), "r"(cnt)
                                 : "memory");
                }
                off = __shfl_sync(0xffffffffu, off, 0);
                // predicated stores and reductions: no divergent branch per descriptor
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const bool p = (mw[u] >> lane) & 1u;
                    blk_sts_if(p, list_s + 4u * (uint32_t)(off + __popc(mw[u] & lt)), (uint32_t)x[u]);
                    blk_red_add_if(p, bins_s + 4u * ((uint32_t)x[u] >> sh), 1u);
                    off += __popc(mw[u]);
                }
            }
            __syncthreads();
        }
        const int ne = *count;
        // ---- bin counts -> ends of the bins (thread t: bins [t*per, t*per+per))
        {
            const int b0 = tid * per, b1 = min(g.nbins, b0 + per);
            int run = 0;
            for (int b = b0; b < b1; ++b) run += bins[b];
            int tot;
            int acc = blk_scan(run, L.wt, tot);
            for (int b = b0; b < b1; ++b) {  // exclusive starts (cursors for the scatter)
                const int c = bins[b];
                bins[b] = acc;
                acc += c;
            }
        }
        __syncthreads();
        for (int e = tid; e < ne; e += NT) {
            const int32_t x = list[e];
            buf[atomicAdd(&bins[x >> sh], 1)] = x;  // bins[b] ends as the end of bin b
        }
        __syncthreads();
        // ---- sort every bin (thread per bin): its ids go to [start, end) of the row.  Bins
        // hold ~2-4 ids: an 8-wide bitonic network in registers, 16-wide for the rare bins of
        // 9-16 ids, a rank loop beyond (never at the default geometry).  The network replaced
        // a rank-by-comparison loop per id (38% of the kernel's instructions at config 3).
        for (int b = tid; b < g.nbins; b += NT) {
            const int bl = b > 0 ? bins[b - 1] : 0, bh = bins[b], k = bh - bl;
            if (k == 0) continue;
            if (k <= 8) {
                bins_sort_out<8, OutT, COMPACT>(buf + bl, k, orow + bl, compact, pol_out);
            } else if (k <= 16) {
                bins_sort_out<16, OutT, COMPACT>(buf + bl, k, orow + bl, compact, pol_out);
            } else {
                for (int p = bl; p < bh; ++p) {
                    const int32_t x = buf[p];
                    int r = bl;
                    for (int q = bl; q < bh; ++q) r += buf[q] < x;
                    stg_pol(orow + r, COMPACT ? __ldg(compact + x) : x, pol_out);
                }
            }
        }
        __syncthreads();
        for (int b = tid; b < g.nbins; b += NT) bins[b] = 0;
        // (the next row's slot pass ends with a barrier before the bins are counted again)
    }
}

template <typename OutT, bool COMPACT>
int run_bins(const RowArgs &a, const BinArgs &g, int sms, cudaStream_t s) {
    const size_t smem = bins_smem_bytes(g);
    auto kern = k_fill_bins<OutT, COMPACT>;
    allow_max_smem(kern);
    prefer_max_shared(kern);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, g.threads, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms, rows));
    kern<<<(unsigned)grid, g.threads, smem, s>>>(a, g);
    return 1;
}

}  // namespace

size_t blk_smem_bytes(const BlkArgs &g, int groups) {
    (void)groups;
    return (size_t)g.nga * 16 + (size_t)((g.nga + 1) & ~1) * 4 + (size_t)((g.threads + 1) & ~1) * 4 +
           (size_t)((g.ecap + 1) & ~1) * 4 + (size_t)g.dcap * 8 +
           (size_t)g.lcap * 12 + 96 * 4;
}

// Geometry: `threads` per CTA (multiple of 32), G groups of 128 ids per thread (power of two
// <= 16); the window is threads*G*128 ids.  Default: 128 threads (measured best at 100k ids:
// 128x8 1.37 ms, 96x16 1.45, 256x4 1.68, 512x2 2.56) and the smallest G covering n, windows
// beyond 256K ids.
void blk_geometry(int64_t n, int threads, int groups, BlkArgs *g) {
    const int nt = threads > 0 ? threads : 128;
    int G = groups;
    if (G <= 0) {
        G = 1;
        while (G < 16 && (int64_t)nt * G * 128 < n) G <<= 1;
    }
    g->threads = nt;
    g->groups = G;
    const int64_t wb = (int64_t)nt * G * 128;
    g->wb = (int32_t)wb;
    g->nwin = (int32_t)((std::max<int64_t>(n, 1) + wb - 1) / wb);
    // bitmap groups actually touched (the window may be wider than n), whole threads
    const int64_t used = (std::min<int64_t>(std::max<int64_t>(n, 1), wb) + 127) / 128;
    g->nga = (int32_t)((used + G - 1) / G * G);
}

int launch_fill_blk(const RowArgs &a, const BlkArgs &g, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    return out64 ? run_blk_t<int64_t>(a, g, sms, s) : run_blk_t<int32_t>(a, g, sms, s);
}

}  // namespace pcg

namespace pcg {

size_t bins_smem_bytes(const BinArgs &g) {
    return (size_t)g.ecap * 8 + (size_t)((g.nbins + 1) & ~1) * 4 + (size_t)g.dcap * 8 +
           (size_t)g.lcap * 12 + 33 * 4;
}

// bins of 2^shift ids with 2-4 admitted ids per bin on average: shift = floor(log2(4n / mean
// row)).  Measured at 1M ids (~3.1k per row, before the bitonic bin sort): ~4 ids per bin
// 23.7 ms, ~1 id per bin 28.0 ms (more bins: more shared memory, fewer CTAs); with the bin
// sort, double-width bins 22.8 ms and half-width 24.9 vs 20.7 ms.
void bins_geometry(int64_t n, double mean_deg, int threads, BinArgs *g) {
    // ~16 of the row's ids per thread, 64-384 threads.  Measured: 100K ids (2.1k per row) 128
    // threads 1.256 ms, 192 1.37; 1M (3.1k per row) 192 20.7 ms, 128 22.9, 256 23.1; 500k with
    // 8.5k per row 384 36.9 ms, 192 57.7
    const int nt = (int)((mean_deg / 16.0 + 16.0) / 32.0) * 32;
    g->threads = threads > 0 ? threads : std::max(64, std::min(384, nt));
    int sh = 0;
    const double want = mean_deg > 1.0 ? 4.0 * (double)n / mean_deg : (double)n;
    while (sh < 30 && (double)(1LL << (sh + 1)) <= want) ++sh;
    g->shift = sh;
    g->nbins = (int32_t)((std::max<int64_t>(n, 1) + (1LL << sh) - 1) >> sh);
}

int launch_fill_bins(const RowArgs &a, const BinArgs &g, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    const bool c = a.compact != nullptr;
    if (out64) return c ? run_bins<int64_t, true>(a, g, sms, s) : run_bins<int64_t, false>(a, g, sms, s);
    return c ? run_bins<int32_t, true>(a, g, sms, s) : run_bins<int32_t, false>(a, g, sms, s);
}

}  // namespace pcg
