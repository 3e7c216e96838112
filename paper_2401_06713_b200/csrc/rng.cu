// Palette lists on the device: rng.py:22-70 + driver.py:175-188, bit-identical.
//   key_v   = mix64(v * phi + mix64(seed + phi * iteration))        (stream_keys)
//   draw_k  = mix64(key_v + (k+1) * phi)                             (draws)
//   Floyd:  for step k, j = P - L + k: t = draw_k % (j+1); take t unless already taken, else j
//   rows sorted ascending, + palette_base                            (sample_distinct)
// One thread per vertex; the <= L picks so far are checked linearly (L is ~20-60).
#include "pcg_internal.cuh"

namespace pcg {
namespace {

constexpr uint64_t PHI = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

template <int LMAX>
__global__ void k_assign_lists(const int64_t *__restrict__ active, int64_t n, uint64_t base_key,
                               int64_t P, int L, int64_t palette_base, int64_t *__restrict__ out) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint64_t key = mix64((uint64_t)active[i] * PHI + base_key);
    int64_t pick[LMAX];
    for (int k = 0; k < L; ++k) {
        const uint64_t j = (uint64_t)(P - L + k);
        uint64_t t = mix64(key + (uint64_t)(k + 1) * PHI) % (j + 1);
        bool taken = false;
        for (int x = 0; x < k; ++x) taken |= (uint64_t)pick[x] == t;
        if (taken) t = j;
        // insertion into the sorted prefix
        int x = k;
        while (x > 0 && pick[x - 1] > (int64_t)t) {
            pick[x] = pick[x - 1];
            --x;
        }
        pick[x] = (int64_t)t;
    }
    int64_t *row = out + i * L;
    for (int k = 0; k < L; ++k) row[k] = pick[k] + palette_base;
}

}  // namespace

int launch_assign_lists(const int64_t *active, int64_t n, uint64_t base_key, int64_t P, int L,
                        int64_t palette_base, int64_t *out, cudaStream_t s) {
    if (n == 0) return 0;
    const int tb = 128;
    const unsigned grid = (unsigned)((n + tb - 1) / tb);
    if (L <= 32) k_assign_lists<32><<<grid, tb, 0, s>>>(active, n, base_key, P, L, palette_base, out);
    else if (L <= 128) k_assign_lists<128><<<grid, tb, 0, s>>>(active, n, base_key, P, L, palette_base, out);
    else k_assign_lists<1024><<<grid, tb, 0, s>>>(active, n, base_key, P, L, palette_base, out);
    return 1;
}

}  // namespace pcg
