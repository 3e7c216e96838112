// K1 — the commuting-pair count over the whole upper triangle (view_edges_scanned,
// conflict.py:78,115; predicate pauli.py:258-268 / graph.py:335-336).
//
// Every unordered pair needs its parity bit  parity(popc(A_i & B_j)), so this is a GF(2)
// matrix product A * B^T whose 1-bits we count.  Two kernels:
//
//  * k_commute_direct — 128x128 upper-triangle tiles staged in shared memory; each thread
//    owns 8x8 pairs: kw LOP3 + 1 POPC per pair, parities collected 32 at a time with a
//    funnel shift and counted with one more POPC.  Bound: POPC/LOP3 issue (~13-16
//    pairs/clk/SM).
//
//  * k_commute_fr — "four Russians" (M4RM): for a j-block of 1024 partners the CTA builds,
//    for every 4-bit slice g of the K-bit vector, the 16 XOR-combinations of the 4
//    transposed partner bit-rows (one 32-bit word per lane = 32 partners).  A row i then
//    costs one shared-memory lookup per 4-bit slice per 32 partners: K/4 LDS.32 + K/8 LOP3
//    per 1024 pairs per warp.  Table layout puts lane t's entry in bank t, and the lookup
//    index is warp-uniform (same i), so every LDS is a single conflict-free wavefront.  The
//    per-row lookup offsets are precomputed once (k_fr_prep) as 16-bit words and turned
//    into addresses with one PRMT.  Bound: shared-memory wavefronts (1/clk/SM).
#include <cub/cub.cuh>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

__device__ __forceinline__ void tile_of(int64_t t, int64_t T, int64_t &bi, int64_t &bj) {
    // row-major upper triangle: S(b) = b*T - b*(b-1)/2 tiles precede row b
    const double a = 2.0 * (double)T + 1.0;
    int64_t b = (int64_t)((a - sqrt(a * a - 8.0 * (double)t)) * 0.5);
    if (b < 0) b = 0;
    if (b > T - 1) b = T - 1;
    auto S = [T](int64_t r) { return r * T - r * (r - 1) / 2; };
    while (b > 0 && S(b) > t) --b;
    while (b + 1 < T && S(b + 1) <= t) ++b;
    bi = b;
    bj = b + (t - S(b));
}

template <int KW>
__global__ void __launch_bounds__(256) k_commute_direct(const uint32_t *__restrict__ A,
                                                        const uint32_t *__restrict__ B,
                                                        int64_t T, int64_t tile0, int64_t tile1,
                                                        unsigned long long *__restrict__ anti) {
    __shared__ uint32_t As[K1_TILE * KW];
    __shared__ uint32_t Bs[K1_TILE * KW];
    __shared__ unsigned long long red[8];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    unsigned long long local = 0;
    for (int64_t t = tile0 + blockIdx.x; t < tile1; t += gridDim.x) {
        int64_t bi, bj;
        tile_of(t, T, bi, bj);
        __syncthreads();
        const uint32_t *ga = A + bi * K1_TILE * KW;
        const uint32_t *gb = B + bj * K1_TILE * KW;
        for (int e = threadIdx.x; e < K1_TILE * KW; e += 256) {
            As[e] = __ldg(ga + e);
            Bs[e] = __ldg(gb + e);
        }
        __syncthreads();
        uint32_t a[8][KW];
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int k = 0; k < KW; ++k) a[r][k] = As[(ty + 16 * r) * KW + k];
        const bool diag = (bi == bj);
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            uint32_t bits = 0;
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
                const int c = half * 4 + cc;
                uint32_t b[KW];
#pragma unroll
                for (int k = 0; k < KW; ++k) b[k] = Bs[(tx + 16 * c) * KW + k];
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    uint32_t acc = a[r][0] & b[0];
#pragma unroll
                    for (int k = 1; k < KW; ++k) acc ^= a[r][k] & b[k];
                    uint32_t par = __popc(acc);
                    if (diag && (tx + 16 * c) <= (ty + 16 * r)) par = 0;
                    bits = __funnelshift_r(bits, par, 1);
                }
            }
            local += __popc(bits);
        }
    }
    // block reduction
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

// Generic kw (very long strings): one pair per thread-iteration, same tiling.
__global__ void __launch_bounds__(256) k_commute_generic(const uint32_t *__restrict__ A,
                                                         const uint32_t *__restrict__ B, int kw,
                                                         int64_t T, int64_t tile0, int64_t tile1,
                                                         unsigned long long *__restrict__ anti) {
    __shared__ unsigned long long red[8];
    unsigned long long local = 0;
    for (int64_t t = tile0 + blockIdx.x; t < tile1; t += gridDim.x) {
        int64_t bi, bj;
        tile_of(t, T, bi, bj);
        for (int p = threadIdx.x; p < K1_TILE * K1_TILE; p += 256) {
            const int r = p >> 7, c = p & 127;
            if (bi == bj && c <= r) continue;
            const uint32_t *a = A + (bi * K1_TILE + r) * kw;
            const uint32_t *b = B + (bj * K1_TILE + c) * kw;
            uint32_t acc = 0;
            for (int k = 0; k < kw; ++k) acc ^= __ldg(a + k) & __ldg(b + k);
            local += __popc(acc) & 1u;
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < 8; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

// ---------------------------------------------------------------------------------------
// Four-Russians kernel.
// ---------------------------------------------------------------------------------------
constexpr int FR_WARPS = 16;

// H[i] holds, for every 4-bit slice g of A_i, the 16-bit table row  h = (g>>1)*16 + v_g,
// two slices per word (g even in the low half).
template <int KW>
__global__ void k_fr_prep(const uint32_t *__restrict__ A, int64_t npad, uint32_t *__restrict__ H) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= npad) return;
    const uint32_t *a = A + i * KW;
    uint32_t *h = H + i * (KW * 4);
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        const uint32_t w = a[k];
#pragma unroll
        for (int m = 0; m < 4; ++m) {  // 8 slices per word -> 4 output words
            const int g = k * 8 + 2 * m;
            const uint32_t v0 = (w >> (8 * m)) & 15u, v1 = (w >> (8 * m + 4)) & 15u;
            const uint32_t base = (uint32_t)(g >> 1) * 16u;
            h[k * 4 + m] = (base + v0) | ((base + v1) << 16);
        }
    }
}

template <int KW>
__global__ void __launch_bounds__(FR_WARPS * 32) k_commute_fr(
    const uint32_t *__restrict__ B, const uint32_t *__restrict__ H, int64_t n,
    const int64_t *__restrict__ item_start, int64_t njb, int32_t ichunk, int64_t item0,
    int64_t item1, unsigned long long *__restrict__ anti) {
    constexpr int K = 32 * KW;           // bits per vector
    constexpr int NG = K / 4;            // 4-bit slices
    constexpr int TBL_WORDS = NG * 16 * 32;
    constexpr int BT_STRIDE = K + 1;     // padded row of the transposed block
    extern __shared__ __align__(16) uint32_t smem[];
    uint32_t *tbl = smem;                      // TBL_WORDS
    uint32_t *bt = smem + TBL_WORDS;           // 32 * BT_STRIDE
    __shared__ unsigned long long red[FR_WARPS];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lb0 = (uint32_t)lane * 4u, lb1 = 128u + (uint32_t)lane * 4u;
    const char *tb = reinterpret_cast<const char *>(tbl);

    // contiguous item range of this CTA (tables reused while the j-block repeats)
    const int64_t nitems = item1 - item0;
    const int64_t my0 = item0 + nitems * blockIdx.x / gridDim.x;
    const int64_t my1 = item0 + nitems * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_jb = -1;
    unsigned long long local = 0;

    for (int64_t it = my0; it < my1; ++it) {
        // item -> (jb, ic): item_start is the exclusive prefix of items per j-block
        int64_t lo = 0, hi = njb;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (item_start[mid] <= it) lo = mid; else hi = mid;
        }
        const int64_t jb = lo, ic = it - item_start[jb];
        if (jb != cur_jb) {
            __syncthreads();  // previous tables no longer in use
            // phase A: transpose the 1024 partner vectors into bit rows bt[t][k]
            for (int t = warp; t < 32; t += FR_WARPS) {
                const uint32_t *bj = B + (jb * K1_FR_JB + 32 * t + lane) * KW;
                uint32_t v[KW];
#pragma unroll
                for (int k = 0; k < KW; ++k) v[k] = __ldg(bj + k);
#pragma unroll
                for (int k = 0; k < KW; ++k) {
                    uint32_t mine = 0;
#pragma unroll
                    for (int s = 0; s < 32; ++s) {
                        const uint32_t word = __ballot_sync(0xffffffffu, (v[k] >> s) & 1u);
                        if (lane == s) mine = word;
                    }
                    bt[t * BT_STRIDE + 32 * k + lane] = mine;
                }
            }
            __syncthreads();
            // phase B: 16 XOR combinations per slice, entry (g, v, t) at word
            // ((g>>1)*16 + v)*64 + (g&1)*32 + t
            for (int g = warp; g < NG; g += FR_WARPS) {
                const uint32_t *row = bt + lane * BT_STRIDE + 4 * g;
                const uint32_t b0 = row[0], b1 = row[1], b2 = row[2], b3 = row[3];
                uint32_t *dst = tbl + (g >> 1) * 16 * 64 + (g & 1) * 32 + lane;
#pragma unroll
                for (int v = 0; v < 16; ++v) {
                    uint32_t e = 0;
                    if (v & 1) e ^= b0;
                    if (v & 2) e ^= b1;
                    if (v & 4) e ^= b2;
                    if (v & 8) e ^= b3;
                    dst[v * 64] = e;
                }
            }
            __syncthreads();
            cur_jb = jb;
        }
        const int64_t jlast = min(n, (jb + 1) * (int64_t)K1_FR_JB);  // exclusive
        const int64_t i0 = ic * ichunk;
        const int64_t i1 = min(i0 + ichunk, jlast);
        const int64_t jbase = jb * K1_FR_JB + 32 * lane;
        for (int64_t i = i0 + warp; i < i1; i += FR_WARPS) {
            const uint4 *hp = reinterpret_cast<const uint4 *>(H + i * (KW * 4));
            uint32_t acc = 0;
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                const uint4 hv = __ldg(hp + k);
                const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    const uint32_t ad0 = __byte_perm(hw[m], lb0, 0x5104);
                    const uint32_t ad1 = __byte_perm(hw[m], lb1, 0x5324);
                    acc ^= *reinterpret_cast<const uint32_t *>(tb + ad0) ^
                           *reinterpret_cast<const uint32_t *>(tb + ad1);
                }
            }
            // partners j = jbase + s with j > i (padding rows j >= n have parity 0)
            uint32_t mask;
            const int64_t d = i - jbase;
            if (d < 0) mask = 0xffffffffu;
            else if (d >= 31) mask = 0u;
            else mask = ~((2u << d) - 1u);
            local += __popc(acc & mask);
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < FR_WARPS; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

// ---------------------------------------------------------------------------------------
// Four-Russians kernel, wide entries: a 2048-partner j-block, lane t owns partners
// 64t..64t+63 and every table entry is 64-bit (two 32-partner words).  One LDS.64 + one
// PRMT per 4-bit slice per 2048 pairs per warp: half the shared-memory instructions and
// address computations of the 32-bit layout for the same wavefronts (the 32-bit kernel is
// bound by LSU instruction issue — mio_throttle — at ~54% of the shared wavefront peak).
// Entry (g, v, t) lives at byte (g>>1)*8192 + ((v<<1)|(g&1))*256 + t*8: the slice-pair
// offset is an LDS immediate (unrolled g), the rest is one PRMT of the row's precomputed
// byte ((v<<1)|(g&1)) (k_fr_prep2) with the lane's t*8.
// ---------------------------------------------------------------------------------------
template <int KW>
__global__ void k_fr_prep2(const uint32_t *__restrict__ A, int64_t npad, uint32_t *__restrict__ H) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= npad) return;
    const uint32_t *a = A + i * KW;
    uint32_t *h = H + i * (KW * 4);
#pragma unroll
    for (int k = 0; k < KW; ++k) {
        const uint32_t w = a[k];
#pragma unroll
        for (int m = 0; m < 4; ++m) {  // slices g = 8k+2m (low half) and 8k+2m+1 (high half)
            const uint32_t v0 = (w >> (8 * m)) & 15u, v1 = (w >> (8 * m + 4)) & 15u;
            h[k * 4 + m] = ((v0 << 1) << 8) | ((((v1 << 1) | 1u) << 8) << 16);
        }
    }
}

template <int KW>
__global__ void __launch_bounds__(FR_WARPS * 32) k_commute_fr2(
    const uint32_t *__restrict__ B, const uint32_t *__restrict__ H, int64_t n,
    const int64_t *__restrict__ item_start, int64_t njb, int32_t ichunk, int64_t item0,
    int64_t item1, unsigned long long *__restrict__ anti) {
    constexpr int K = 32 * KW;           // bits per vector
    constexpr int NG = K / 4;            // 4-bit slices
    constexpr int JB = 2048;
    constexpr int TBL_BYTES = (NG / 2) * 8192;
    constexpr int BT_STRIDE = K + 1;     // padded row of the transposed block
    extern __shared__ __align__(16) uint32_t smem[];
    char *tbl = reinterpret_cast<char *>(smem);
    uint32_t *bt = smem + TBL_BYTES / 4;       // 64 * BT_STRIDE
    __shared__ unsigned long long red[FR_WARPS];

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lb = (uint32_t)lane * 8u;
    const uint32_t tbl_s = (uint32_t)__cvta_generic_to_shared(tbl);

    const int64_t nitems = item1 - item0;
    const int64_t my0 = item0 + nitems * blockIdx.x / gridDim.x;
    const int64_t my1 = item0 + nitems * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_jb = -1;
    unsigned long long local = 0;

    for (int64_t it = my0; it < my1; ++it) {
        int64_t lo = 0, hi = njb;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (item_start[mid] <= it) lo = mid; else hi = mid;
        }
        const int64_t jb = lo, ic = it - item_start[jb];
        if (jb != cur_jb) {
            __syncthreads();  // previous tables no longer in use
            // phase A: transpose the 2048 partner vectors into bit rows bt[t][k], t = 32-group
            for (int t = warp; t < 64; t += FR_WARPS) {
                const uint32_t *bj = B + (jb * JB + 32 * t + lane) * KW;
                uint32_t v[KW];
#pragma unroll
                for (int k = 0; k < KW; ++k) v[k] = __ldg(bj + k);
#pragma unroll
                for (int k = 0; k < KW; ++k) {
                    uint32_t mine = 0;
#pragma unroll
                    for (int s = 0; s < 32; ++s) {
                        const uint32_t word = __ballot_sync(0xffffffffu, (v[k] >> s) & 1u);
                        if (lane == s) mine = word;
                    }
                    bt[t * BT_STRIDE + 32 * k + lane] = mine;
                }
            }
            __syncthreads();
            // phase B: 16 XOR combinations per slice; lane t builds the entry of groups 2t, 2t+1
            for (int g = warp; g < NG; g += FR_WARPS) {
                const uint32_t *r0 = bt + (2 * lane) * BT_STRIDE + 4 * g;
                const uint32_t *r1 = r0 + BT_STRIDE;
                const uint32_t a0 = r0[0], a1 = r0[1], a2 = r0[2], a3 = r0[3];
                const uint32_t c0 = r1[0], c1 = r1[1], c2 = r1[2], c3 = r1[3];
                char *dst = tbl + (g >> 1) * 8192 + (g & 1) * 256 + lane * 8;
#pragma unroll
                for (int v = 0; v < 16; ++v) {
                    uint32_t e0 = 0, e1 = 0;
                    if (v & 1) { e0 ^= a0; e1 ^= c0; }
                    if (v & 2) { e0 ^= a1; e1 ^= c1; }
                    if (v & 4) { e0 ^= a2; e1 ^= c2; }
                    if (v & 8) { e0 ^= a3; e1 ^= c3; }
                    *reinterpret_cast<uint2 *>(dst + v * 512) = make_uint2(e0, e1);
                }
            }
            __syncthreads();
            cur_jb = jb;
        }
        const int64_t jlast = min(n, (jb + 1) * (int64_t)JB);  // exclusive
        const int64_t i0 = ic * ichunk;
        const int64_t i1 = min(i0 + ichunk, jlast);
        const int64_t jbase = jb * JB + 64 * lane;
        for (int64_t i = i0 + warp; i < i1; i += FR_WARPS) {
            const uint4 *hp = reinterpret_cast<const uint4 *>(H + i * (KW * 4));
            uint32_t acc0 = 0, acc1 = 0;
#pragma unroll
            for (int k = 0; k < KW; ++k) {
                const uint4 hv = __ldg(hp + k);
                const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w};
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    // slices g = 8k+2m and g+1 share the slice pair (g>>1) = 4k+m
                    const uint32_t base = tbl_s + (uint32_t)(4 * k + m) * 8192u;
                    const uint32_t ad0 = base + __byte_perm(hw[m], lb, 0x7614);
                    const uint32_t ad1 = base + __byte_perm(hw[m], lb, 0x7634);
                    uint2 e0, e1;
                    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(e0.x), "=r"(e0.y) : "r"(ad0));
                    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(e1.x), "=r"(e1.y) : "r"(ad1));
                    acc0 ^= e0.x ^ e1.x;
                    acc1 ^= e0.y ^ e1.y;
                }
            }
            // partners j = jbase + s (word 0) and jbase + 32 + s (word 1) with j > i
            const int64_t d0 = i - jbase, d1 = d0 - 32;
            const uint32_t m0 = d0 < 0 ? 0xffffffffu : (d0 >= 31 ? 0u : ~((2u << d0) - 1u));
            const uint32_t m1 = d1 < 0 ? 0xffffffffu : (d1 >= 31 ? 0u : ~((2u << d1) - 1u));
            local += __popc(acc0 & m0) + __popc(acc1 & m1);
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < FR_WARPS; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

// ---------------------------------------------------------------------------------------
// Four-Russians with 6-bit slices (the default for kw 2/4, q <= 64).  The bound of the
// 4-bit kernels is shared-memory bytes per pair: one 8-byte entry per 4-bit slice per 64
// partners = K/32 bytes per pair (4 B at q = 64).  6-bit slices need ceil(K/6) lookups
// instead of K/4 (22 instead of 32 at q = 64: 2.75 B per pair), but a 64-entry table per
// slice is 4x the 16-entry one, so the j-block shrinks to 1024 partners (16 lanes x 64)
// and each half-warp runs its own row: a half-warp reads 16 consecutive 8-byte entries =
// exactly one 128-byte wavefront, still conflict-free.  Tables: ceil(K/6) x 64 entries x
// 128 B = 176 KB at K = 128, plus 16.5 KB for the transposed block; one CTA per SM.
//
// Entry (slice g, value v, half-lane l) at byte g*8192 + v*128 + 8*l: word 0 = the 32
// partners 64l..64l+31, word 1 = 64l+32..64l+63.  The table base is aligned to 8 KB, so a
// lookup address is  base_l | ((A_i >> 6g) & 63) << 7  — one funnel shift and one LOP3
// straight from the row's bits (no per-row offset array), with g*8192 as the immediate.
// ---------------------------------------------------------------------------------------
template <int KW, int RPW>
__global__ void __launch_bounds__(FR_WARPS * 32, 1) k_commute_fr6(
    const uint32_t *__restrict__ A, const uint32_t *__restrict__ B, int64_t n,
    const int64_t *__restrict__ item_start, int64_t njb, int32_t ichunk, int64_t item0,
    int64_t item1, unsigned long long *__restrict__ anti) {
    constexpr int K = 32 * KW;           // bits per vector
    constexpr int NG = (K + 5) / 6;      // 6-bit slices (the last one narrower)
    constexpr int JB = K1_FR_JB;         // 1024 partners
    constexpr int BT_STRIDE = K + 1;
    constexpr int LPR = 32 / RPW;        // lanes per row
    constexpr int EB = 128 / LPR;        // bytes per lane lookup (8: LDS.64, 16: LDS.128)
    constexpr int NW = EB / 4;           // 32-partner words per lane
    extern __shared__ __align__(16) uint32_t smem[];
    __shared__ unsigned long long red[FR_WARPS];
    const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t tbl_s = (smem_s + 8191u) & ~8191u;  // 8 KB aligned table base
    char *tbl = reinterpret_cast<char *>(smem) + (tbl_s - smem_s);
    uint32_t *bt = reinterpret_cast<uint32_t *>(tbl + NG * 8192);  // 32 x BT_STRIDE

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / LPR, hl = lane % LPR;
    const uint32_t base_l = tbl_s + (uint32_t)(hl * EB);

    const int64_t nitems = item1 - item0;
    const int64_t my0 = item0 + nitems * blockIdx.x / gridDim.x;
    const int64_t my1 = item0 + nitems * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_jb = -1;
    unsigned long long local = 0;

    for (int64_t it = my0; it < my1; ++it) {
        int64_t lo = 0, hi = njb;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (item_start[mid] <= it) lo = mid; else hi = mid;
        }
        const int64_t jb = lo, ic = it - item_start[jb];
        if (jb != cur_jb) {
            __syncthreads();  // previous tables no longer in use
            // phase A: transpose the 1024 partner vectors into bit rows bt[t][k], t = 32-group
            for (int t = warp; t < 32; t += FR_WARPS) {
                const uint32_t *bj = B + (jb * JB + 32 * t + lane) * KW;
                uint32_t v[KW];
#pragma unroll
                for (int k = 0; k < KW; ++k) v[k] = __ldg(bj + k);
#pragma unroll
                for (int k = 0; k < KW; ++k) {
                    uint32_t mine = 0;
#pragma unroll
                    for (int s = 0; s < 32; ++s) {
                        const uint32_t word = __ballot_sync(0xffffffffu, (v[k] >> s) & 1u);
                        if (lane == s) mine = word;
                    }
                    bt[t * BT_STRIDE + 32 * k + lane] = mine;
                }
            }
            __syncthreads();
            // phase B: the 64 XOR combinations of each slice's 6 bit rows; warp g-slice, lane
            // t = 32-partner group t (byte 4t of the 128-byte entry)
            for (int g = warp; g < NG; g += FR_WARPS) {
                const uint32_t *row = bt + lane * BT_STRIDE + 6 * g;
                uint32_t r[6];
#pragma unroll
                for (int b = 0; b < 6; ++b) r[b] = (6 * g + b < K) ? row[b] : 0u;
                uint32_t *dst = reinterpret_cast<uint32_t *>(tbl + g * 8192) + lane;
#pragma unroll 8
                for (int v = 0; v < 64; ++v) {
                    uint32_t e = 0;
#pragma unroll
                    for (int b = 0; b < 6; ++b) e ^= (v >> b & 1) ? r[b] : 0u;
                    dst[v * 32] = e;
                }
            }
            __syncthreads();
            cur_jb = jb;
        }
        const int64_t jlast = min(n, (jb + 1) * (int64_t)JB);  // exclusive
        const int64_t i0 = ic * ichunk;
        const int64_t i1 = min(i0 + ichunk, jlast);
        const int64_t jbase = jb * JB + 32 * NW * hl;
        for (int64_t i = i0 + RPW * warp + grp; i < i1; i += RPW * FR_WARPS) {
            uint32_t a[KW + 1];
            if constexpr (KW == 4) {
                const uint4 av = __ldg(reinterpret_cast<const uint4 *>(A + i * 4));
                a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
            } else {
                const uint2 av = __ldg(reinterpret_cast<const uint2 *>(A + i * 2));
                a[0] = av.x; a[1] = av.y;
            }
            a[KW] = 0u;
            uint32_t acc[NW];
#pragma unroll
            for (int w = 0; w < NW; ++w) acc[w] = 0u;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const int o = 6 * g, w = o >> 5, sh = o & 31;
                // bits o..o+5 of the row, already shifted to bit 7 (the entry stride)
                uint32_t x;
                if (sh + 6 <= 32) x = sh >= 7 ? (a[w] >> (sh - 7)) : (a[w] << (7 - sh));
                else x = __funnelshift_r(a[w], a[w + 1], sh) << 7;
                uint32_t ad;  // (x & 0x1f80) | base_l: one LOP3 (base_l has no bits in 7..12)
                asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(ad) : "r"(x), "r"(0x1f80u), "r"(base_l));
                ad += (uint32_t)(g * 8192);
                if constexpr (NW == 4) {
                    uint32_t e0, e1, e2, e3;
                    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                                 : "=r"(e0), "=r"(e1), "=r"(e2), "=r"(e3) : "r"(ad));
                    acc[0] ^= e0; acc[1] ^= e1; acc[2] ^= e2; acc[3] ^= e3;
                } else {
                    uint32_t e0, e1;
                    asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(e0), "=r"(e1) : "r"(ad));
                    acc[0] ^= e0; acc[1] ^= e1;
                }
            }
            // partners j = jbase + 32w + s with j > i
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const int64_t d = i - (jbase + 32 * w);
                const uint32_t m = d < 0 ? 0xffffffffu : (d >= 31 ? 0u : ~((2u << d) - 1u));
                local += __popc(acc[w] & m);
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < FR_WARPS; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

template <typename K>
int occupancy_grid(K kernel, int threads, size_t smem, int sms, int64_t work) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int64_t g = (int64_t)per_sm * sms;
    if (g > work) g = work;
    return (int)(g < 1 ? 1 : g);
}

template <int KW>
int run_direct(const uint32_t *A, const uint32_t *B, int64_t T, int64_t t0, int64_t t1,
               unsigned long long *anti, int sms, cudaStream_t s) {
    const int grid = occupancy_grid(k_commute_direct<KW>, 256, 0, sms, t1 - t0);
    k_commute_direct<KW><<<grid, 256, 0, s>>>(A, B, T, t0, t1, anti);
    return 1;
}

template <int KW>
size_t fr_smem() {
    return (size_t)(KW * 32 / 4) * 16 * 32 * 4 + (size_t)32 * (KW * 32 + 1) * 4;
}

template <int KW>
size_t fr2_smem() {
    return (size_t)(KW * 32 / 4 / 2) * 8192 + (size_t)64 * (KW * 32 + 1) * 4;
}

template <int KW>
int run_fr2(const uint32_t *B, const uint32_t *H, int64_t n, const int64_t *item_start,
            int64_t njb, int32_t ichunk, int64_t item0, int64_t item1,
            unsigned long long *anti, int sms, cudaStream_t s) {
    const size_t smem = fr2_smem<KW>();
    allow_max_smem(k_commute_fr2<KW>);
    const int grid = occupancy_grid(k_commute_fr2<KW>, FR_WARPS * 32, smem, sms, item1 - item0);
    k_commute_fr2<KW><<<grid, FR_WARPS * 32, smem, s>>>(B, H, n, item_start, njb, ichunk, item0,
                                                       item1, anti);
    return 1;
}

template <int KW>
size_t fr6_smem() {
    constexpr int K = 32 * KW, NG = (K + 5) / 6;
    return 8192 + (size_t)NG * 8192 + (size_t)32 * (K + 1) * 4;  // + alignment slack
}

template <int KW, int RPW>
int run_fr6(const uint32_t *A, const uint32_t *B, int64_t n, const int64_t *item_start,
            int64_t njb, int32_t ichunk, int64_t item0, int64_t item1,
            unsigned long long *anti, int sms, cudaStream_t s) {
    const size_t smem = fr6_smem<KW>();
    allow_max_smem(k_commute_fr6<KW, RPW>);
    const int grid = occupancy_grid(k_commute_fr6<KW, RPW>, FR_WARPS * 32, smem, sms, item1 - item0);
    k_commute_fr6<KW, RPW><<<grid, FR_WARPS * 32, smem, s>>>(A, B, n, item_start, njb, ichunk,
                                                            item0, item1, anti);
    return 1;
}

template <int KW>
int run_fr(const uint32_t *B, const uint32_t *H, int64_t n, const int64_t *item_start,
           int64_t njb, int32_t ichunk, int64_t item0, int64_t item1,
           unsigned long long *anti, int sms, cudaStream_t s) {
    const size_t smem = fr_smem<KW>();
    allow_max_smem(k_commute_fr<KW>);
    const int grid = occupancy_grid(k_commute_fr<KW>, FR_WARPS * 32, smem, sms, item1 - item0);
    k_commute_fr<KW><<<grid, FR_WARPS * 32, smem, s>>>(B, H, n, item_start, njb, ichunk, item0,
                                                      item1, anti);
    return 1;
}

}  // namespace

int launch_commute_direct(const uint32_t *A, const uint32_t *B, int32_t kw, int64_t npad,
                          int64_t tile0, int64_t tile1, unsigned long long *anti, int sms,
                          cudaStream_t s) {
    if (tile1 <= tile0) return 0;
    const int64_t T = npad / K1_TILE;
    switch (kw) {
        case 2: return run_direct<2>(A, B, T, tile0, tile1, anti, sms, s);
        case 4: return run_direct<4>(A, B, T, tile0, tile1, anti, sms, s);
        case 6: return run_direct<6>(A, B, T, tile0, tile1, anti, sms, s);
        case 8: return run_direct<8>(A, B, T, tile0, tile1, anti, sms, s);
        case 10: return run_direct<10>(A, B, T, tile0, tile1, anti, sms, s);
        case 12: return run_direct<12>(A, B, T, tile0, tile1, anti, sms, s);
        default: {
            const int grid = occupancy_grid(k_commute_generic, 256, 0, sms, tile1 - tile0);
            k_commute_generic<<<grid, 256, 0, s>>>(A, B, kw, T, tile0, tile1, anti);
            return 1;
        }
    }
}

bool fr_supported(int32_t kw) { return kw == 2 || kw == 4 || kw == 6 || kw == 8; }

int fr_jb(int32_t kw, int wide) { return (wide && (kw == 2 || kw == 4)) ? K1_FR_JB2 : K1_FR_JB; }

int launch_commute_fr6_items(const uint32_t *A, const uint32_t *B, int32_t kw, int64_t n,
                             const int64_t *item_start, int64_t njb, int32_t ichunk,
                             int64_t item0, int64_t item1, unsigned long long *anti, int sms,
                             int wide_loads, cudaStream_t s) {
    if (item1 <= item0) return 0;
    if (wide_loads) {  // LDS.128, a quarter-warp per row
        switch (kw) {
            case 2: return run_fr6<2, 4>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
            case 4: return run_fr6<4, 4>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
            default: return 0;
        }
    }
    switch (kw) {  // LDS.64, a half-warp per row
        case 2: return run_fr6<2, 2>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        case 4: return run_fr6<4, 2>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        default: return 0;
    }
}

int launch_fr_prep2(const uint32_t *A, int32_t kw, int64_t npad, uint32_t *H, cudaStream_t s) {
    const int tb = 256;
    const unsigned grid = (unsigned)((npad + tb - 1) / tb);
    switch (kw) {
        case 2: k_fr_prep2<2><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        case 4: k_fr_prep2<4><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        default: return 0;
    }
}

int launch_commute_fr2_items(const uint32_t *B, const uint32_t *H, int32_t kw, int64_t n,
                             const int64_t *item_start, int64_t njb, int32_t ichunk,
                             int64_t item0, int64_t item1, unsigned long long *anti, int sms,
                             cudaStream_t s) {
    if (item1 <= item0) return 0;
    switch (kw) {
        case 2: return run_fr2<2>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        case 4: return run_fr2<4>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        default: return 0;
    }
}

int launch_fr_prep(const uint32_t *A, int32_t kw, int64_t npad, uint32_t *H, cudaStream_t s) {
    const int tb = 256;
    const unsigned grid = (unsigned)((npad + tb - 1) / tb);
    switch (kw) {
        case 2: k_fr_prep<2><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        case 4: k_fr_prep<4><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        case 6: k_fr_prep<6><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        case 8: k_fr_prep<8><<<grid, tb, 0, s>>>(A, npad, H); return 1;
        default: return 0;
    }
}

int launch_commute_fr_items(const uint32_t *B, const uint32_t *H, int32_t kw, int64_t n,
                            const int64_t *item_start, int64_t njb, int32_t ichunk,
                            int64_t item0, int64_t item1, unsigned long long *anti, int sms,
                            cudaStream_t s) {
    if (item1 <= item0) return 0;
    switch (kw) {
        case 2: return run_fr<2>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        case 4: return run_fr<4>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        case 6: return run_fr<6>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        case 8: return run_fr<8>(B, H, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
        default: return 0;
    }
}

}  // namespace pcg
