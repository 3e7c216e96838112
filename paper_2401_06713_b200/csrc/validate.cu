// GPU exhaustive validator: properness of a coloring of a Pauli view, the
// exhaustive mode of validation.validate (/root/reference/pkg/src/palettecolor/validation.py:63-82)
// without its 20,000-vertex cap (graph.py:34).
//
// A violation is a commuting pair (a G' edge) whose endpoints share a color, so it can only
// occur inside a color class.  The active vertices are sorted by color (stable: a class lists
// its vertices in ascending local index), and every vertex checks its class successors with
// the same predicate as the builder, parity(popc(A_i & B_j)) == 0.  Work is sum over classes
// of |class|^2 / 2 predicate evaluations (tiny for a proper coloring; quadratic only for a
// degenerate one).  The first `cap` violations in the reference's enumeration order (i
// ascending, then j ascending; graph.py:379-407) are produced exactly: per-row counts, an
// exclusive scan over rows, and an emit pass for the rows whose offset is below the cap.
// |E| (oracle_edges) is the builder's commuting-pair sweep (K1) over the same view.
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

__global__ void k_class_keys(const int64_t *__restrict__ color, int64_t n, int64_t *__restrict__ keys,
                             int32_t *__restrict__ vals) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t c = color[i];
    keys[i] = c == INT64_MIN ? INT64_MAX : c;  // uncolored vertices sort last, never checked
    vals[i] = (int32_t)i;
}

__device__ __forceinline__ bool commute_pair(const uint32_t *__restrict__ A,
                                             const uint32_t *__restrict__ B, int32_t kw,
                                             int32_t i, int32_t j) {
    uint32_t acc = 0u;
    for (int k = 0; k < kw; ++k) acc ^= __ldg(A + (int64_t)i * kw + k) & __ldg(B + (int64_t)j * kw + k);
    return (__popc(acc) & 1u) == 0u;
}

template <bool EMIT>
__global__ void k_class_pairs(const int64_t *__restrict__ keys, const int32_t *__restrict__ vals,
                              int64_t n, const uint32_t *__restrict__ A,
                              const uint32_t *__restrict__ B, int32_t kw,
                              int64_t *__restrict__ cnt, const int64_t *__restrict__ off,
                              int64_t cap, int64_t *__restrict__ pairs) {
    const int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t key = keys[p];
    const int32_t i = vals[p];
    if (key == INT64_MAX) {
        if (!EMIT) cnt[i] = 0;
        return;
    }
    int64_t o = EMIT ? off[i] : 0;
    if (EMIT && o >= cap) return;
    int64_t c = 0;
    for (int64_t q = p + 1; q < n && keys[q] == key; ++q) {
        const int32_t j = vals[q];
        if (commute_pair(A, B, kw, i, j)) {
            if (EMIT) {
                pairs[2 * o] = i;
                pairs[2 * o + 1] = j;
                if (++o >= cap) return;
            } else {
                ++c;
            }
        }
    }
    if (!EMIT) cnt[i] = c;
}

}  // namespace

int launch_class_keys(const int64_t *color, int64_t n, int64_t *keys, int32_t *vals, cudaStream_t s) {
    if (n == 0) return 0;
    k_class_keys<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(color, n, keys, vals);
    return 1;
}

int launch_class_pairs(bool emit, const int64_t *keys, const int32_t *vals, int64_t n,
                       const uint32_t *A, const uint32_t *B, int32_t kw, int64_t *cnt,
                       const int64_t *off, int64_t cap, int64_t *pairs, cudaStream_t s) {
    if (n == 0) return 0;
    const unsigned grid = (unsigned)((n + 127) / 128);
    if (emit)
        k_class_pairs<true><<<grid, 128, 0, s>>>(keys, vals, n, A, B, kw, cnt, off, cap, pairs);
    else
        k_class_pairs<false><<<grid, 128, 0, s>>>(keys, vals, n, A, B, kw, cnt, off, cap, pairs);
    return 1;
}

}  // namespace pcg
