// Input preparation kernels (K0): Pauli words -> bit-plane vectors, color lists -> int32
// relative ids + per-entry row ids (input of the color-bucket index).
//
// Bilinear form.  The reference tests anticommutation as parity(popcount(w_i & w_j)) over
// the 3-bit codes X=110, Y=101, Z=011, I=000 (pauli.py:7-14, 258-268).  For valid codes that
// parity equals the symplectic form  <x_i,z_j> + <z_i,x_j>  (mod 2) with x_p = code bit 2
// and z_p = code bit 0, so each vertex gets
//     A_i = [x_i | z_i]     B_j = [z_j | x_j]        (each plane ceil(q/32) uint32 words)
// and every kernel evaluates parity(popc(A_i & B_j)) — 2*ceil(q/32) words instead of
// ceil(3q/32).  If any code is invalid (only possible when a caller builds a PauliSet by
// hand), the context re-encodes with A = B = the raw 3-bit words, which is the reference
// predicate verbatim.
#include "pcg_internal.cuh"

namespace pcg {

namespace {

__device__ __forceinline__ uint32_t code_at(const uint64_t *w, int nwords, int p) {
    const int bit = 3 * p;
    const int wi = bit >> 6, off = bit & 63;
    uint64_t v = w[wi] >> off;
    if (off > 61 && wi + 1 < nwords) v |= w[wi + 1] << (64 - off);
    return static_cast<uint32_t>(v & 7u);
}

// One thread per local vertex; rows [n, npad) are zero padding (parity 0 with everything).
__global__ void k_encode(const uint64_t *__restrict__ words, int nwords,
                         const int64_t *__restrict__ active, int64_t n, int64_t npad, int q,
                         int raw, uint32_t *__restrict__ A, uint32_t *__restrict__ B, int kw,
                         int32_t *__restrict__ bad) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= npad) return;
    uint32_t *a = A + i * kw, *b = B + i * kw;
    if (i >= n) {
        for (int k = 0; k < kw; ++k) a[k] = b[k] = 0u;
        return;
    }
    const uint64_t *w = words + active[i] * nwords;
    if (raw) {
        for (int k = 0; k < kw; ++k) {
            const int wi = k >> 1;
            const uint32_t v = wi < nwords ? static_cast<uint32_t>(w[wi] >> (32 * (k & 1))) : 0u;
            a[k] = b[k] = v;
        }
        return;
    }
    const int qw = kw >> 1;
    bool invalid = false;
    for (int t = 0; t < qw; ++t) {
        uint32_t xw = 0u, zw = 0u;
        const int p0 = t * 32;
        const int pe = min(q, p0 + 32);
        for (int p = p0; p < pe; ++p) {
            const uint32_t c = code_at(w, nwords, p);
            // valid codes: 000 (I), 110 (X), 101 (Y), 011 (Z)
            invalid |= (c == 1u) | (c == 2u) | (c == 4u) | (c == 7u);
            xw |= ((c >> 2) & 1u) << (p - p0);
            zw |= (c & 1u) << (p - p0);
        }
        a[t] = xw;
        a[qw + t] = zw;
        b[t] = zw;
        b[qw + t] = xw;
    }
    // trailing stream bits beyond 3q must be zero (pauli.py:13-14)
    const int tail = 3 * q;
    const int wi = tail >> 6, off = tail & 63;
    if (wi < nwords) {
        uint64_t rest = off ? (w[wi] >> off) : w[wi];
        if (rest) invalid = true;
        for (int k = wi + 1; k < nwords; ++k)
            if (w[k]) invalid = true;
    }
    if (invalid) atomicExch(bad, 1);
}

// One thread per list entry: relative color (int32) and the entry's row.
__global__ void k_lists(const int64_t *__restrict__ lists, const int64_t *__restrict__ loff,
                        int64_t n, int L, int64_t entries, int64_t base, int64_t P,
                        int32_t *__restrict__ lrel, int32_t *__restrict__ row_of,
                        int32_t *__restrict__ bad) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e >= entries) return;
    const int64_t rel = lists[e] - base;
    if (rel < 0 || rel >= P) atomicOr(bad, 2);
    lrel[e] = static_cast<int32_t>(rel < 0 || rel >= P ? 0 : rel);
    int64_t r;
    if (loff == nullptr) {
        r = e / L;
    } else {  // ragged: binary search the row whose range holds e
        int64_t lo = 0, hi = n;
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (loff[mid] <= e) lo = mid; else hi = mid;
        }
        r = lo;
    }
    row_of[e] = static_cast<int32_t>(r);
}

// bstart[c] = first position of color c in the sorted color array (lower bound), c in [0,P]:
// one thread per sorted entry writes the starts of the colors between its predecessor's color
// and its own (coalesced; no search).  A color listed twice in one row shows up as two
// adjacent entries of one bucket with the same row (the sort is stable in entry order): flag 4.
__global__ void k_bucket_bounds(const int32_t *__restrict__ sorted, const int32_t *__restrict__ eidx,
                                const int32_t *__restrict__ row_of, int64_t entries, int64_t P,
                                int32_t *__restrict__ bstart, int32_t *__restrict__ bad) {
    const int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (e > entries) return;
    const int64_t prev = e > 0 ? sorted[e - 1] : -1;
    const int64_t cur = e < entries ? sorted[e] : P + 1;
    for (int64_t c = prev + 1; c <= cur && c <= P; ++c) bstart[c] = static_cast<int32_t>(e);
    if (e > 0 && e < entries && prev == cur && row_of[eidx[e]] == row_of[eidx[e - 1]])
        atomicOr(bad, 4);
}

}  // namespace

int launch_encode(const uint64_t *words, int32_t nwords, const int64_t *active, int64_t n,
                  int64_t npad, int32_t q, int raw, uint32_t *A, uint32_t *B, int32_t kw,
                  int32_t *bad, cudaStream_t s) {
    if (npad == 0) return 0;
    const int tb = 256;
    k_encode<<<(unsigned)((npad + tb - 1) / tb), tb, 0, s>>>(words, nwords, active, n, npad, q,
                                                             raw, A, B, kw, bad);
    return 1;
}

int launch_lists(const int64_t *lists, const int64_t *loff, int64_t n, int32_t L,
                 int64_t entries, int64_t base, int64_t P, int32_t *lrel, int32_t *row_of,
                 int32_t *bad, cudaStream_t s) {
    if (entries == 0) return 0;
    const int tb = 256;
    k_lists<<<(unsigned)((entries + tb - 1) / tb), tb, 0, s>>>(lists, loff, n, L, entries, base,
                                                               P, lrel, row_of, bad);
    return 1;
}

int launch_bucket_bounds(const int32_t *sorted_colors, const int32_t *eidx, const int32_t *row_of,
                         int64_t entries, int64_t P, int32_t *bstart, int32_t *bad, cudaStream_t s) {
    const int tb = 256;
    k_bucket_bounds<<<(unsigned)((entries + 1 + tb - 1) / tb), tb, 0, s>>>(sorted_colors, eidx, row_of,
                                                                         entries, P, bstart, bad);
    return 1;
}

}  // namespace pcg
