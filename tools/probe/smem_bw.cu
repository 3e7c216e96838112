// Shared-memory load throughput on this GPU (the K1 bound): bytes per clock per SM for
// conflict-free table lookups of the shapes the four-Russians kernels use.
//   v2_half : LDS.64, each half-warp reads 16 consecutive 8-byte entries of its own row
//             (k_commute_fr6: 1024-partner tables)
//   v2_warp : LDS.64, the whole warp reads 32 consecutive 8-byte entries (k_commute_fr2)
//   v4_quarter: LDS.128, each quarter-warp reads 8 consecutive 16-byte entries
//   v1_warp : LDS.32, the whole warp reads 32 consecutive words (k_commute_fr)
// Row indices are pseudo-random per (row group, step) from a register xorshift, as data-
// dependent lookups are in K1.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 smem_bw.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int TBL = 160 * 1024;
constexpr int STEPS = 4096;

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned *out, long long *cycles) {
    extern __shared__ __align__(16) unsigned char sm[];
    for (int i = threadIdx.x; i < TBL / 4; i += blockDim.x) reinterpret_cast<unsigned *>(sm)[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    unsigned x = 0x9E3779B9u * (threadIdx.x / (MODE == 0 ? 16 : MODE == 2 ? 8 : 32) + 1) + blockIdx.x;
    unsigned acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    long long t0 = clock64();
#pragma unroll 1
    for (int s = 0; s < STEPS; s += 16) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            x += 0x9E3779B9u * (u + 1);  // independent addresses within the batch
            if (MODE == 0) {  // half-warp rows of 128 B
                const unsigned ad = base + ((x & 1023u) << 7) + (lane & 15) * 8;
                unsigned a, b;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(ad));
                acc0 ^= a; acc1 ^= b;
            } else if (MODE == 1) {  // warp rows of 256 B
                const unsigned ad = base + ((x & 511u) << 8) + lane * 8;
                unsigned a, b;
                asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(a), "=r"(b) : "r"(ad));
                acc0 ^= a; acc1 ^= b;
            } else if (MODE == 2) {  // quarter-warp rows of 128 B, 16-byte entries
                const unsigned ad = base + ((x & 1023u) << 7) + (lane & 7) * 16;
                unsigned a, b, c, d;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(ad));
                acc0 ^= a; acc1 ^= b; acc2 ^= c; acc3 ^= d;
            } else {  // warp rows of 128 B, 4-byte entries
                const unsigned ad = base + ((x & 1023u) << 7) + lane * 4;
                unsigned a;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(a) : "r"(ad));
                acc0 ^= a;
            }
        }
    }
    long long t1 = clock64();
    if ((acc0 ^ acc1 ^ acc2 ^ acc3) == 0x12345678u) out[0] = 1;
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char *name, int threads, int bytes_per_lane) {
    unsigned *out;
    long long *cyc;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaMalloc(&cyc, sms * 8);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, TBL);
    k<MODE><<<sms, threads, TBL>>>(out, cyc);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<MODE><<<sms, threads, TBL>>>(out, cyc);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    long long c[256];
    cudaMemcpy(c, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double cmax = 0;
    for (int i = 0; i < sms; ++i) cmax = c[i] > cmax ? c[i] : cmax;
    const double bytes_sm = (double)threads * STEPS * bytes_per_lane;
    printf("%-11s threads %4d: %.1f B/clk/SM (%.3f ms, %.2f TB/s over %d SMs)\n", name, threads,
           bytes_sm / cmax, ms, bytes_sm * sms / (ms * 1e-3) / 1e12, sms);
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    for (int t : {256, 512}) {
        run<0>("v2_half", t, 8);
        run<1>("v2_warp", t, 8);
        run<2>("v4_quarter", t, 16);
        run<3>("v1_warp", t, 4);
    }
    return 0;
}
