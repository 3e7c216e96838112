// Host memory write bandwidth probe (diagnostic for the e2e path): streaming-store fill and
// int32 -> int64 widen with N OpenMP threads, 4K pages vs madvise(MADV_HUGEPAGE).
#include <immintrin.h>
#include <omp.h>
#include <sys/mman.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <initializer_list>
#include <algorithm>
static double now() { return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count(); }
__attribute__((target("avx512f"))) static void widen(int64_t *to, const int32_t *from, size_t len) {
    size_t x = 0;
    for (; x < len && (reinterpret_cast<uintptr_t>(to + x) & 63); ++x) to[x] = from[x];
    for (; x + 16 <= len; x += 16) {
        __m256i a = _mm256_loadu_si256((const __m256i *)(from + x));
        __m256i b = _mm256_loadu_si256((const __m256i *)(from + x + 8));
        _mm512_stream_si512((__m512i *)(to + x), _mm512_cvtepi32_epi64(a));
        _mm512_stream_si512((__m512i *)(to + x + 8), _mm512_cvtepi32_epi64(b));
    }
    for (; x < len; ++x) to[x] = from[x];
    _mm_sfence();
}
int main() {
    const size_t N = 207513882;
    for (int huge = 0; huge < 2; ++huge) {
        size_t bytes = ((N * 8 + (2 << 20) - 1) / (2 << 20)) * (2 << 20);
        int64_t *dst = (int64_t *)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (huge) madvise(dst, bytes, MADV_HUGEPAGE);
        memset(dst, 1, bytes);
        int32_t *src = (int32_t *)aligned_alloc(64, ((N * 4 + 63) / 64) * 64);
        for (size_t i = 0; i < N; ++i) src[i] = (int32_t)i;
        for (int T : {4, 8, 16}) {
            double best = 1e9;
            for (int r = 0; r < 3; ++r) {
                double t0 = now();
#pragma omp parallel for num_threads(T) schedule(static)
                for (int t = 0; t < T; ++t) {
                    size_t a = N * t / T, b = N * (t + 1) / T;
                    widen(dst + a, src + a, b - a);
                }
                best = std::min(best, now() - t0);
            }
            printf("huge=%d threads=%2d widen int32->int64: %.1f ms  %.1f GB/s written\n", huge, T, best * 1e3, N * 8 / best / 1e9);
        }
        free(src);
        munmap(dst, bytes);
    }
    return 0;
}
