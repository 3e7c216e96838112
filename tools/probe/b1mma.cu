// Throughput probe: mma.sync m16n8k256 b1 (AND + POPC) on sm_100a, 8 independent chains/warp.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k(uint32_t *out, int iters) {
    uint32_t a0 = threadIdx.x * 2654435761u, a1 = a0 ^ 0x9e3779b9u, a2 = a0 + 7, a3 = a0 * 3;
    uint32_t b0 = a0 ^ 0x85ebca6bu, b1 = a1 + 11;
    int c[8][4] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ch = 0; ch < 8; ++ch) {
            asm volatile(
                "mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc "
                "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                : "+r"(c[ch][0]), "+r"(c[ch][1]), "+r"(c[ch][2]), "+r"(c[ch][3])
                : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
        }
        a0 += 1; b0 ^= it;
    }
    int s = 0;
    for (int ch = 0; ch < 8; ++ch) s += c[ch][0] + c[ch][1] + c[ch][2] + c[ch][3];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint32_t *out; cudaMalloc(&out, 1 << 24);
    for (int warps : {4, 8, 16}) {
        const int iters = 4096, blocks = sms * 2;
        k<<<blocks, warps * 32>>>(out, 16);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k<<<blocks, warps * 32>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double mmas = (double)blocks * warps * iters * 8;
        const double per_sm_per_ns = mmas / sms / (ms * 1e6);
        printf("warps/block %2d x2 blocks/SM: %.3f ms  %.3e mma/s  %.3f mma/clk/SM (at 1.965 GHz)  "
               "-> %.1f Tbitop/s\n", warps, ms, mmas / (ms * 1e-3), per_sm_per_ns / 1.965,
               mmas / (ms * 1e-3) * 16 * 8 * 256 * 2 / 1e12);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
