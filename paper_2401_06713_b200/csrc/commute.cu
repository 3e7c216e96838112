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
//  * the four-Russians kernel with 8-bit slices, k_commute_fr8 (commute8.cu), is the default
//    for q <= 128; this file keeps the direct kernel as the path for wider vectors and as an
//    independent cross-check in the parity tests (k1_algo 1).  The 4-, 5- and 6-bit
//    four-Russians kernels of rounds 1-2 were measured slower than the 8-bit one and removed.
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

}  // namespace pcg
