// Delta encoding of the conflict CSR for the device->host copy of the public build.
//
// The host API returns int64 neighbor ids (conflict.py:148-161), so the host must write 8
// bytes per CSR entry; at config 2 (207M entries) the copy-out is bound by host memory
// traffic, not by PCIe.  Rows are strictly ascending, so an entry is sent as its gap to the
// previous entry of the row (the first entry: its value + 1): one byte when the gap is below
// 255, else the escape byte 255 and the full id in an exception list (row-major order).  PCIe
// carries ~1 byte per entry instead of 4, and the host reads 1 byte per 8 it writes.  Sparse
// rows (mean gap above 64 ids, e.g. 1M ids with ~3k neighbors) use 16-bit gaps (escape 65535)
// instead: bytes would escape a large share of the entries.
//
//   k_delta_count : warp per row — gap bytes, exceptions per row
//   (exclusive scan of the per-row exception counts, CUB)
//   k_delta_exc   : warp per row — the exceptions of the row, in entry order (ballot ranks)
#include <cub/cub.cuh>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

template <bool WRITE, typename G>
__global__ void k_delta(const int32_t *__restrict__ nbr, const int64_t *__restrict__ rowoff,
                        int64_t rows, G *__restrict__ bytes, int32_t *__restrict__ xcount,
                        const int64_t *__restrict__ xoff, int32_t *__restrict__ xval) {
    constexpr uint32_t ESC = sizeof(G) == 1 ? 255u : 65535u;
    const int lane = threadIdx.x & 31;
    const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w; r < rows; r += nw) {
        const int64_t b = rowoff[r], e = rowoff[r + 1];
        int cnt = 0;
        int64_t xo = WRITE ? xoff[r] : 0;
        for (int64_t x0 = b; x0 < e; x0 += 32) {
            const int64_t x = x0 + lane;
            uint32_t gap = 0u;
            int32_t v = 0;
            if (x < e) {
                v = nbr[x];
                gap = x == b ? (uint32_t)v + 1u : (uint32_t)(v - nbr[x - 1]);
            }
            const bool esc = x < e && gap >= ESC;
            const uint32_t bal = __ballot_sync(0xffffffffu, esc);
            if (!WRITE) {
                if (x < e) bytes[x] = esc ? (G)ESC : (G)gap;
                cnt += __popc(bal);
            } else {
                if (esc) xval[xo + __popc(bal & ((1u << lane) - 1u))] = v;
                xo += __popc(bal);
            }
        }
        if (!WRITE && lane == 0) xcount[r] = cnt;
    }
}

}  // namespace

// int32 -> int64 widen of a CSR slice (chunks the pipelined copy-out ships as int64 by DMA)
__global__ void k_widen(const int32_t *__restrict__ src, int64_t *__restrict__ dst, int64_t count) {
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < count;
         x += (int64_t)gridDim.x * blockDim.x)
        dst[x] = src[x];
}

int launch_widen(const int32_t *src, int64_t *dst, int64_t count, int sms, cudaStream_t s) {
    if (count <= 0) return 0;
    const int64_t grid = std::min<int64_t>((count + 255) / 256, (int64_t)sms * 8);
    k_widen<<<(unsigned)grid, 256, 0, s>>>(src, dst, count);
    return 1;
}

int launch_delta(bool write, bool wide, const int32_t *nbr, const int64_t *rowoff, int64_t rows,
                 void *bytes, int32_t *xcount, const int64_t *xoff, int32_t *xval, int sms,
                 cudaStream_t s) {
    if (rows <= 0) return 0;
    const int64_t grid = std::min<int64_t>((rows + 7) / 8, (int64_t)sms * 16);
    uint8_t *b8 = static_cast<uint8_t *>(bytes);
    uint16_t *b16 = static_cast<uint16_t *>(bytes);
    if (write && wide)
        k_delta<true, uint16_t><<<(unsigned)grid, 256, 0, s>>>(nbr, rowoff, rows, b16, xcount, xoff, xval);
    else if (write)
        k_delta<true, uint8_t><<<(unsigned)grid, 256, 0, s>>>(nbr, rowoff, rows, b8, xcount, xoff, xval);
    else if (wide)
        k_delta<false, uint16_t><<<(unsigned)grid, 256, 0, s>>>(nbr, rowoff, rows, b16, xcount, xoff, xval);
    else
        k_delta<false, uint8_t><<<(unsigned)grid, 256, 0, s>>>(nbr, rowoff, rows, b8, xcount, xoff, xval);
    return 1;
}

}  // namespace pcg
