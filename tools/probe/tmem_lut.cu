// Can tensor memory serve as a second lookup-table store next to shared memory (K1)?
// Measures, per SM, the throughput of data-dependent (warp-uniform column) TMEM reads
// (tcgen05.ld.32x32b.x1: 32 lanes x 4 B = 128 B per warp instruction) alone, shared-memory
// LDS.128 quarter-warp lookups alone (the k_commute_fr6 pattern), and both at once in one CTA
// (half the warps each).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tmem_lut.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TBL = 160 * 1024;
constexpr int STEPS = 8192;
constexpr int WARPS = 32;

__device__ __forceinline__ uint32_t tld(uint32_t taddr) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr));
    return v;
}

// MODE 0: TMEM only (all warps); 1: smem only (all warps); 2: half/half
// warps [0, nt) read TMEM, warps [nt, ns) read shared memory, the rest idle
template <int MODE>
__global__ void __launch_bounds__(WARPS * 32, 1) k(unsigned *out, long long *cycles, int *bytes, int nt, int ns) {
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < TBL / 4; i += blockDim.x) reinterpret_cast<unsigned *>(sm)[i] = i * 2654435761u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&tbase)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tbase;
    const uint32_t lane_base = tb + ((uint32_t)(32 * (warp & 3)) << 16);
    // fill our quadrant's 512 columns
    if (warp < 4) {
        for (int c = 0; c < 512; ++c) {
            const uint32_t v = (uint32_t)(c * 977 + lane * 131);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(lane_base + c), "r"(v));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const bool use_tmem = warp < nt;
    const int steps = warp < ns ? STEPS : 0;  // idle warps skip the loop
    unsigned x = 0x9E3779B9u * (warp * 4 + (use_tmem ? 0 : (lane >> 3)) + 1) + blockIdx.x;
    unsigned acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
    const unsigned base = (unsigned)__cvta_generic_to_shared(sm);
    __syncthreads();
    long long t0 = clock64();
    int nb = 0;
#pragma unroll 1
    for (int s = 0; s < steps; s += 16) {
        x ^= x << 13; x ^= x >> 17; x ^= x << 5;
        if (use_tmem) {
            uint32_t v[16];
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint32_t col = (x + 0x9E3779B9u * (u + 1)) >> 23;  // warp-uniform, 0..511
                v[u] = tld(lane_base + col);
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int u = 0; u < 16; ++u) acc0 ^= v[u];
            nb += 16 * 128;
        } else {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const unsigned xx = x + 0x9E3779B9u * (u + 1);
                const unsigned ad = base + ((xx & 1023u) << 7) + (lane & 7) * 16;
                unsigned a, b, c, d;
                asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(ad));
                acc0 ^= a; acc1 ^= b; acc2 ^= c; acc3 ^= d;
            }
            nb += 16 * 512;
        }
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 ^ acc1 ^ acc2 ^ acc3;
    __syncthreads();
    if (lane == 0) {
        atomicAdd(bytes + 2 * blockIdx.x + (use_tmem ? 0 : 1), nb);
        if (steps) atomicMax(reinterpret_cast<unsigned long long *>(cycles + blockIdx.x), (unsigned long long)(t1 - t0));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int MODE>
void run(const char *name, int sms, int nt, int ns) {
    unsigned *out;
    long long *cyc;
    int *bytes;
    cudaMalloc(&out, (size_t)sms * WARPS * 32 * 4);
    cudaMalloc(&cyc, sms * 8);
    cudaMalloc(&bytes, sms * 8);
    cudaMemset(cyc, 0, sms * 8);
    cudaMemset(bytes, 0, sms * 8);
    cudaFuncSetAttribute(k<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, TBL);
    k<MODE><<<sms, WARPS * 32, TBL>>>(out, cyc, bytes, nt, ns);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("%s: %s\n", name, cudaGetErrorString(e)); return; }
    cudaMemset(cyc, 0, sms * 8);
    cudaMemset(bytes, 0, sms * 8);
    k<MODE><<<sms, WARPS * 32, TBL>>>(out, cyc, bytes, nt, ns);
    cudaDeviceSynchronize();
    long long c[256];
    int b[512];
    cudaMemcpy(c, cyc, sms * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(b, bytes, sms * 8, cudaMemcpyDeviceToHost);
    double st = 0, ss = 0;
    for (int i = 0; i < sms; ++i) { st += (double)b[2 * i] / (double)c[i]; ss += (double)b[2 * i + 1] / (double)c[i]; }
    st /= sms; ss /= sms;
    printf("%-10s tmem warps %2d smem warps %2d: tmem %6.1f + smem %6.1f = %6.1f B/clk/SM; K1 q=64 pairs/clk "
           "(tmem 4 B/pair, smem 2.75 B/pair) %5.1f\n", name, nt, ns - nt, st, ss, st + ss, st / 4 + ss / 2.75);
    cudaFree(out); cudaFree(cyc); cudaFree(bytes);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int cfg[][2] = {{0, 16}, {16, 32}, {12, 32}, {8, 32}, {8, 24}, {4, 20}, {12, 28}, {20, 32}};
    for (auto &c : cfg) run<0>("lookups", sms, c[0], c[1]);
    return 0;
}
