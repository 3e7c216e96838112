// K2 — conflict rows.  For every row i of the build, the admitted partners
//     { j != i : list(i) ∩ list(j) != ∅  and  parity(popc(A_i & B_j)) == 0 }
// (conflict.py:72-78: edge & (mask_i & mask_j).any()), produced in ascending j, i.e.
// directly in the canonical CSR row order of conflict.py:148-161 — no sort pass.
//
// Exact list intersection without the reference's dense ceil(P/64)-word masks: the
// candidates of row i are the union of its L color buckets (bucket c = ascending local ids
// holding color c).  One warp per row:
//   mark   — lanes walk the L buckets (one bucket per lane, 4 loads in flight) and set
//            bits in a per-warp shared-memory bitmap covering a window of `window` ids;
//            duplicates (pairs sharing several colors) collapse in the bitmap.
//   test   — lane l owns a contiguous segment of the window; it queues its set bits and
//            tests them 8 at a time (8 independent partner loads in flight): commute
//            predicate parity(popc(A_i & B_j)).
//   emit   — count pass: degree and upper degree (j > i).  Fill pass: admitted bits are
//            written back into the bitmap, a warp exclusive scan of the lane counts gives
//            each lane's output offset, and lanes write their ids in order.
// Windows advance left to right, so rows come out sorted.  Rows are independent: the
// multi-GPU path simply gives each GPU a row range.
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

constexpr int RW_WARPS = 8;
constexpr int QLEN = 8;

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

template <int KW, bool FILL, typename OutT>
__global__ void __launch_bounds__(RW_WARPS * 32) k_rows(RowArgs a) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int WW = a.window >> 5;  // bitmap words
    const int SPL = WW >> 5;       // words per lane segment (multiple of 4)
    const int slots = (2 * a.slot_cap + 3) & ~3;  // keep every warp region 16-byte aligned
    uint32_t *bm = smem + (size_t)warp * (WW + QLEN * 32 + slots);
    int32_t *q = reinterpret_cast<int32_t *>(bm + WW);
    int32_t *cur = q + QLEN * 32;
    int32_t *cend = cur + a.slot_cap;
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    __syncwarp();

    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int64_t stride = (int64_t)gridDim.x * RW_WARPS;
    for (int64_t i = a.row_begin + (int64_t)blockIdx.x * RW_WARPS + warp; i < a.row_end;
         i += stride) {
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
            // ---- mark the candidates of this window
            for (int s = lane; s < Li; s += 32) {
                int p = cur[s];
                const int e = cend[s];
                while (p < e) {
                    int m[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) m[u] = (p + u < e) ? __ldg(a.bmem + p + u) : INT_MAX;
                    int k = 0;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        if (m[u] < w1) {
                            const int off = m[u] - w0;
                            atomicOr(&bm[off >> 5], 1u << (off & 31));
                            ++k;
                        }
                    p += k;
                    if (k < 4) break;
                }
                cur[s] = p;
            }
            __syncwarp();
            if (lane == 0 && self >= w0 && self < w1) {
                const int off = self - w0;
                atomicAnd(&bm[off >> 5], ~(1u << (off & 31)));
            }
            __syncwarp();

            // ---- test this lane's segment
            const int seg0 = lane * SPL;
            int nq = 0, lane_adm = 0;
            auto flush = [&](int cntq) {
                uint32_t par[QLEN];
                int offs[QLEN];
#pragma unroll
                for (int k = 0; k < QLEN; ++k) {
                    offs[k] = k < cntq ? q[k * 32 + lane] : 0;
                    par[k] = k < cntq ? ai.parity(a.B, w0 + offs[k], a.kw) : 1u;
                }
#pragma unroll
                for (int k = 0; k < QLEN; ++k) {
                    if (k < cntq && par[k] == 0u) {
                        ++lane_adm;
                        if constexpr (FILL) {
                            bm[offs[k] >> 5] |= 1u << (offs[k] & 31);
                        } else {
                            ++cnt;
                            cntu += (w0 + offs[k] > self) ? 1 : 0;
                        }
                    }
                }
            };
            for (int t = 0; t < SPL; t += 4) {
                uint4 *p4 = reinterpret_cast<uint4 *>(bm + seg0 + t);
                const uint4 v = *p4;
                if ((v.x | v.y | v.z | v.w) == 0u) continue;
                *p4 = make_uint4(0u, 0u, 0u, 0u);
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t wd = wv[u];
                    while (wd) {
                        const int b = __ffs(wd) - 1;
                        wd &= wd - 1u;
                        q[nq * 32 + lane] = ((seg0 + t + u) << 5) | b;
                        if (++nq == QLEN) {
                            flush(QLEN);
                            nq = 0;
                        }
                    }
                }
            }
            if (nq) flush(nq);

            if constexpr (FILL) {
                int total;
                const int base = warp_excl_scan(lane_adm, lane, total);
                int64_t pos = outpos + base;
                for (int t = 0; t < SPL; t += 4) {
                    uint4 *p4 = reinterpret_cast<uint4 *>(bm + seg0 + t);
                    const uint4 v = *p4;
                    if ((v.x | v.y | v.z | v.w) == 0u) continue;
                    *p4 = make_uint4(0u, 0u, 0u, 0u);
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint32_t wd = wv[u];
                        while (wd) {
                            const int b = __ffs(wd) - 1;
                            wd &= wd - 1u;
                            const int32_t j = w0 + (((seg0 + t + u) << 5) | b);
                            out[pos++] = (OutT)(a.compact ? a.compact[j] : j);
                        }
                    }
                }
                outpos += total;
            }
            __syncwarp();
        }
        if constexpr (!FILL) {
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                cnt += __shfl_down_sync(0xffffffffu, cnt, o);
                cntu += __shfl_down_sync(0xffffffffu, cntu, o);
            }
            if (lane == 0) {
                a.deg[i] = cnt;
                a.degu[i] = cntu;
            }
        }
        __syncwarp();
    }
}

template <int KW, bool FILL, typename OutT>
int run_rows(const RowArgs &a, int sms, cudaStream_t s) {
    const size_t per_warp = (size_t)((a.window >> 5) + QLEN * 32 + ((2 * a.slot_cap + 3) & ~3)) * 4;
    const size_t smem = per_warp * RW_WARPS;
    cudaFuncSetAttribute(k_rows<KW, FILL, OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rows<KW, FILL, OutT>,
                                                  RW_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    int64_t grid = (int64_t)per_sm * sms;
    const int64_t need = (rows + RW_WARPS - 1) / RW_WARPS;
    if (grid > need) grid = need;
    if (grid < 1) grid = 1;
    k_rows<KW, FILL, OutT><<<(unsigned)grid, RW_WARPS * 32, smem, s>>>(a);
    return 1;
}

template <bool FILL, typename OutT>
int dispatch_kw(const RowArgs &a, int sms, cudaStream_t s) {
    switch (a.kw) {
        case 2: return run_rows<2, FILL, OutT>(a, sms, s);
        case 4: return run_rows<4, FILL, OutT>(a, sms, s);
        case 6: return run_rows<6, FILL, OutT>(a, sms, s);
        case 8: return run_rows<8, FILL, OutT>(a, sms, s);
        case 12: return run_rows<12, FILL, OutT>(a, sms, s);
        default: return run_rows<0, FILL, OutT>(a, sms, s);
    }
}

__global__ void k_compact(const int32_t *__restrict__ deg, int64_t n,
                          const int32_t *__restrict__ compact, const int64_t *__restrict__ rowoff,
                          const int64_t *__restrict__ active, int64_t *__restrict__ members,
                          int64_t *__restrict__ offsets) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int d = deg[i];
    const int64_t k = compact ? compact[i] : i;
    if (d > 0) {
        members[k] = active[i];
        offsets[k] = rowoff[i];
    }
    if (i == n - 1) offsets[k + (d > 0 ? 1 : 0)] = rowoff[n];
}

}  // namespace

int launch_rows(const RowArgs &a, bool fill, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    if (!fill) return dispatch_kw<false, int32_t>(a, sms, s);
    if (out64) return dispatch_kw<true, int64_t>(a, sms, s);
    return dispatch_kw<true, int32_t>(a, sms, s);
}

int launch_compact(const int32_t *deg, int64_t n, const int32_t *compact, const int64_t *rowoff,
                   const int64_t *active, int64_t *members_out, int64_t *offsets_out,
                   cudaStream_t s) {
    if (n == 0) return 0;
    const int tb = 256;
    k_compact<<<(unsigned)((n + tb - 1) / tb), tb, 0, s>>>(deg, n, compact, rowoff, active,
                                                           members_out, offsets_out);
    return 1;
}

}  // namespace pcg
