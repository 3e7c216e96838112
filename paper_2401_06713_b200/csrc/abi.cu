// C ABI of the B200 conflict-graph builder (include/picasso_b200.h).
//
// Host orchestration of one build, mirroring palettecolor.conflict.build
// (conflict.py:89-167): stage inputs (K0), count (K1 + K2 count), let the caller check
// the budget, then fill (compaction + K2 fill) straight into the caller's buffers.
#include <cub/cub.cuh>

#include <omp.h>

#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "pcg_internal.cuh"

namespace pcg {

cudaError_t ensure(DevBuf &b, size_t bytes) {
    if (bytes == 0) bytes = 16;
    if (b.cap >= bytes) return cudaSuccess;
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
    size_t want = bytes + bytes / 8;  // headroom for slightly larger next builds
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        e = cudaMalloc(&b.p, bytes);
        if (e != cudaSuccess) {
            cudaGetLastError();
            b.p = nullptr;
            return e;
        }
        want = bytes;
    }
    b.cap = want;
    return cudaSuccess;
}

void release(DevBuf &b) {
    if (b.p) cudaFree(b.p);
    b.p = nullptr;
    b.cap = 0;
}

namespace {

struct DegPositive {
    const int32_t *d;
    int64_t n;
    __host__ __device__ int32_t operator()(int64_t i) const { return (i < n && d[i] > 0) ? 1 : 0; }
};
struct DegAt {
    const int32_t *d;
    int64_t n;
    __host__ __device__ int64_t operator()(int64_t i) const { return i < n ? (int64_t)d[i] : 0; }
};

__global__ void k_sum_degrees(const int32_t *__restrict__ deg, const int32_t *__restrict__ degu,
                              int64_t r0, int64_t r1, unsigned long long *out) {
    unsigned long long s = 0, su = 0, m = 0, mx = 0;
    for (int64_t i = r0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < r1;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int d = deg[i];
        s += d;
        su += degu[i];
        m += d > 0;
        mx = d > (int)mx ? (unsigned long long)d : mx;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xffffffffu, s, o);
        su += __shfl_down_sync(0xffffffffu, su, o);
        m += __shfl_down_sync(0xffffffffu, m, o);
        const unsigned long long y = __shfl_down_sync(0xffffffffu, mx, o);
        mx = y > mx ? y : mx;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out + 1, s);
        atomicAdd(out + 2, su);
        atomicAdd(out + 3, m);
        atomicMax(out + 4, mx);
    }
}

int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

}  // namespace
}  // namespace pcg

using namespace pcg;

#define PCG_TRY_CUDA(ctx, expr)                                                      \
    do {                                                                            \
        cudaError_t _e = (expr);                                                    \
        if (_e != cudaSuccess) {                                                    \
            (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(_e);        \
            return _e == cudaErrorMemoryAllocation ? PCG_E_OOM : PCG_E_CUDA;        \
        }                                                                           \
    } while (0)

#define PCG_ALLOC(ctx, buf, bytes)                                                   \
    do {                                                                            \
        cudaError_t _e = ensure((buf), (bytes));                                    \
        if (_e != cudaSuccess) {                                                    \
            (ctx)->err = std::string("device allocation of ") +                     \
                         std::to_string((size_t)(bytes)) + " bytes failed: " +      \
                         cudaGetErrorString(_e);                                    \
            return PCG_E_OOM;                                                       \
        }                                                                           \
    } while (0)

#define PCG_CHECK_LAUNCH(ctx) PCG_TRY_CUDA(ctx, cudaGetLastError())

static int fail(pcg_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return code;
}

extern "C" {

int pcg_version(void) { return 1; }

// why the last pcg_create failed (pcg_last_error(NULL)), per host thread
static thread_local std::string g_create_err = "null context";

int pcg_create(int device, pcg_ctx **out) {
    if (!out) return PCG_E_ARG;
    *out = nullptr;
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess || device < 0 || device >= ndev) {
        g_create_err = e != cudaSuccess ? std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e)
                                        : "device " + std::to_string(device) + " of " +
                                              std::to_string(ndev);
        cudaGetLastError();
        return PCG_E_CUDA;
    }
    pcg_ctx *ctx = new pcg_ctx();
    ctx->device = device;
    e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        g_create_err = std::string("device ") + std::to_string(device) + ": " + cudaGetErrorString(e);
        cudaGetLastError();
        delete ctx;
        return PCG_E_CUDA;
    }
    cudaDeviceGetAttribute(&ctx->sms, cudaDevAttrMultiProcessorCount, device);
    for (auto &e : ctx->ev) cudaEventCreate(&e);
    *out = ctx;
    return PCG_OK;
}

int pcg_destroy(pcg_ctx *ctx) {
    if (!ctx) return PCG_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    DevBuf *bufs[] = {&ctx->words, &ctx->active, &ctx->lists64, &ctx->loff, &ctx->A, &ctx->B,
                      &ctx->lrel, &ctx->rowof, &ctx->keys2, &ctx->vals2, &ctx->bstart,
                      &ctx->cubtmp, &ctx->deg, &ctx->degu, &ctx->compact, &ctx->rowoff,
                      &ctx->scal, &ctx->bad, &ctx->members_o, &ctx->offsets_o, &ctx->nbr_o,
                      &ctx->gdeg, &ctx->items, &ctx->eidx, &ctx->bpos, &ctx->bmemp,
                      &ctx->posof, &ctx->maskoff, &ctx->masks, &ctx->bnd, &ctx->vcolor, &ctx->vkeys,
                      &ctx->vkeys2, &ctx->vvals, &ctx->vvals2, &ctx->vcnt, &ctx->voff,
                      &ctx->vpairs};
    for (DevBuf *b : bufs) release(*b);
    for (auto &m : ctx->xmaps) cudaIpcCloseMemHandle(m.second);
    release(ctx->xbuf);
    release(ctx->workctr);
    for (void *p : ctx->ring)
        if (p) cudaFreeHost(p);
    for (auto &e : ctx->ring_ev) cudaEventDestroy(e);
    for (auto &st : ctx->ring_st) cudaStreamDestroy(st);
    for (auto &e : ctx->chunk_ev) cudaEventDestroy(e);
    if (ctx->k1_stream) cudaStreamDestroy(ctx->k1_stream);
    if (ctx->k1_fork) cudaEventDestroy(ctx->k1_fork);
    if (ctx->k1_done) cudaEventDestroy(ctx->k1_done);
    for (uint8_t *p : ctx->hbytes)
        if (p) cudaFreeHost(p);
    if (ctx->hxval) cudaFreeHost(ctx->hxval);
    if (ctx->hxoff) cudaFreeHost(ctx->hxoff);
    release(ctx->dbytes);
    release(ctx->dxcnt);
    release(ctx->dxoff);
    release(ctx->dxval);
    release(ctx->mrow);
    if (ctx->hs) cudaFreeHost(ctx->hs);
    release(ctx->dwide);
    if (ctx->dma_st) cudaStreamDestroy(ctx->dma_st);
    for (auto &e : ctx->piece_ev) cudaEventDestroy(e);
    if (ctx->scan_ev) cudaEventDestroy(ctx->scan_ev);
    for (auto &hp : ctx->hxpiece)
        if (hp.first) cudaFreeHost(hp.first);
    for (auto &e : ctx->ev)
        if (e) cudaEventDestroy(e);
    for (auto &h : ctx->stage)
        if (h) cudaFreeHost(h);
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return PCG_OK;
}

const char *pcg_last_error(const pcg_ctx *ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int pcg_set_option(pcg_ctx *ctx, const char *key, int64_t value) {
    if (!ctx || !key) return PCG_E_ARG;
    if (!strcmp(key, "k1_algo")) ctx->k1_algo = (int)value;
    else if (!strcmp(key, "window")) ctx->window = (int)value;
    else if (!strcmp(key, "fr_ichunk")) ctx->fr_ichunk = (int)value;
    else if (!strcmp(key, "k2_mode")) ctx->k2_mode = (int)value;
    else if (!strcmp(key, "fill_algo")) ctx->fill_algo = (int)value;
    else if (!strcmp(key, "seg_bits")) ctx->seg_bits = (int)value;
    else if (!strcmp(key, "own_algo")) ctx->own_algo = (int)value;
    else if (!strcmp(key, "own_direct")) ctx->own_direct = (int)value;
    else if (!strcmp(key, "own_bitmap")) ctx->own_bitmap = (int)value;
    else if (!strcmp(key, "d2h_chunk")) ctx->d2h_chunk = (int)value;
    else if (!strcmp(key, "d2h_threads")) ctx->d2h_threads = (int)value;
    else if (!strcmp(key, "d2h_mode")) ctx->d2h_mode = (int)value;
    else if (!strcmp(key, "k1_async")) ctx->k1_async = (int)value;
    else if (!strcmp(key, "own_rows_lo")) ctx->own_lo = value;
    else if (!strcmp(key, "own_rows_hi")) ctx->own_hi = value;
    else if (!strcmp(key, "k1_early")) ctx->k1_early = (int)value;
    else if (!strcmp(key, "d2h_gap16")) ctx->d2h_gap16 = (int)value;
    else if (!strcmp(key, "d2h_pipe")) ctx->d2h_pipe = (int)value;
    else if (!strcmp(key, "d2h_pieces")) ctx->d2h_pieces = (int)value;
    else if (!strcmp(key, "d2h_dma")) ctx->d2h_dma = (int)value;
    else if (!strcmp(key, "blk_threads")) ctx->blk_threads = (int)value;
    else if (!strcmp(key, "blk_groups")) ctx->blk_groups = (int)value;
    else if (!strcmp(key, "blk_dcap")) ctx->blk_dcap = (int)value;
    else if (!strcmp(key, "blk_ecap")) ctx->blk_ecap = (int)value;
    else if (!strcmp(key, "bins_threads")) ctx->bins_threads = (int)value;
    else if (!strcmp(key, "bins_shift")) ctx->bins_shift = (int)value;
    else if (!strcmp(key, "bins_maxdeg")) ctx->bins_maxdeg = (int)value;
    else if (!strcmp(key, "rows_out32")) ctx->rows_out32 = (int)value;
    else if (!strcmp(key, "rows_out_abs")) ctx->rows_out_abs = (int)value;
    else if (!strcmp(key, "dyn_work")) ctx->dyn_work = (int)value;
    else if (!strcmp(key, "fuse_deg")) ctx->fuse_deg = (int)value;
    else if (!strcmp(key, "k1_warps")) ctx->k1_warps = (int)value;
    else if (!strcmp(key, "k1_shard")) ctx->k1_shard = (int)value;
    else if (!strcmp(key, "k1_nshards")) ctx->k1_nshards = (int)std::max<int64_t>(1, value);
    else if (!strcmp(key, "seg_warps")) ctx->seg_warps = (int)value;
    else return fail(ctx, PCG_E_ARG, std::string("unknown option ") + key);
    return PCG_OK;
}

void *pcg_stream(pcg_ctx *ctx) { return ctx ? (void *)ctx->stream : nullptr; }

int pcg_set_profiling(pcg_ctx *ctx, int32_t on) {
    if (!ctx) return PCG_E_ARG;
    ctx->prof = on != 0;
    return PCG_OK;
}

int pcg_kernel_times(pcg_ctx *ctx, float *ms, int32_t n) {
    if (!ctx || !ms) return PCG_E_ARG;
    for (int k = 0; k < n && k < 5; ++k) ms[k] = ctx->ktimes[k];
    return PCG_OK;
}

}  // extern "C"

// --------------------------------------------------------------------------------------
// input staging (K0)
// --------------------------------------------------------------------------------------
static int encode_vectors(pcg_ctx *ctx, bool raw) {
    cudaStream_t s = ctx->stream;
    ctx->raw = raw;
    ctx->kw = raw ? 2 * ctx->nwords : 2 * ((ctx->q + 31) / 32);
    PCG_ALLOC(ctx, ctx->A, (size_t)ctx->npad * ctx->kw * 4);
    PCG_ALLOC(ctx, ctx->B, (size_t)ctx->npad * ctx->kw * 4);
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->bad.p, 0, 8, s));
    launch_encode(ctx->words.as<uint64_t>(), ctx->nwords, ctx->active.as<int64_t>(), ctx->n,
                  ctx->npad, ctx->q, raw ? 1 : 0, ctx->A.as<uint32_t>(), ctx->B.as<uint32_t>(),
                  ctx->kw, ctx->bad.as<int32_t>(), s);
    PCG_CHECK_LAUNCH(ctx);
    return PCG_OK;
}


namespace pcg_prep {
struct PaddedSize {
    const int32_t *bstart;
    int64_t P;
    __host__ __device__ int32_t operator()(int64_t c) const {
        if (c >= P) return 0;
        const int32_t m = bstart[c + 1] - bstart[c];
        return (m + 3) & ~3;
    }
};
struct MaskWords {
    const int32_t *bstart;
    int64_t P;
    __host__ __device__ int64_t operator()(int64_t c) const {
        if (c >= P) return 0;
        const int64_t m = bstart[c + 1] - bstart[c];
        return m * ((m + 31) / 32);
    }
};
__global__ void k_bucket_max(const int32_t *bstart, int64_t P, int32_t *out) {
    int32_t m = 0;
    for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < P;
         c += (int64_t)gridDim.x * blockDim.x)
        m = max(m, bstart[c + 1] - bstart[c]);
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}
__global__ void k_iota(int32_t *x, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i < n) x[i] = (int32_t)i;
}
}  // namespace pcg_prep
using namespace pcg_prep;

// A K1 still running on the side stream reads the bit planes and adds into scal[0]: the main
// stream waits for it before either is rewritten.
static void k1_join(pcg_ctx *ctx) {
    if (ctx->k1_pending && ctx->k1_done) cudaStreamWaitEvent(ctx->stream, ctx->k1_done, 0);
}

// Small device -> host readbacks (sizes, flags, totals) land in pinned scratch: a copy into
// pageable stack memory is a staged, much slower transfer on the critical path of each build.
static unsigned char *pinned_scratch(pcg_ctx *ctx) {
    if (!ctx->hs && cudaHostAlloc(reinterpret_cast<void **>(&ctx->hs), 512, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        ctx->hs = nullptr;
    }
    return ctx->hs;
}

static BucketArgs bucket_args(const pcg_ctx *ctx) {
    BucketArgs b{};
    b.P = ctx->P;
    b.bstart = ctx->bstart.as<int32_t>();
    b.sorted_e = ctx->vals2.as<int32_t>();
    b.row_of = ctx->rowof.as<int32_t>();
    b.bpos = ctx->bpos.as<int32_t>();
    b.maskoff = ctx->maskoff.as<int64_t>();
    b.bmemp = ctx->bmemp.as<int32_t>();
    b.bmem = ctx->masked ? nullptr : ctx->keys2.as<int32_t>();  // keys are dead after bounds
    b.posof = ctx->posof.as<int32_t>();
    b.masks = ctx->masked ? ctx->masks.as<uint32_t>() : nullptr;
    b.A = ctx->A.as<uint32_t>();
    b.B = ctx->B.as<uint32_t>();
    b.kw = ctx->kw;
    return b;
}

static int run_k1(pcg_ctx *ctx, int32_t shard, int32_t nshards, int64_t *pairs, int *launches,
                  cudaStream_t s, unsigned long long *anti);

// K1 launched from the input prep, once the color buckets are sorted (option "k1_early", with
// "k1_async"): the commuting-pair sweep (8 warps per SM) then overlaps the owned masks, the
// count and the fill passes, which take their work from atomic counters (dyn_work) so that
// their CTAs resident next to K1 do the work.  It accumulates into its own counter (scal[7]); the count
// pass of the same build (one shard) takes it over instead of launching K1 again.
static int k1_launch_early(pcg_ctx *ctx, cudaStream_t s) {
    ctx->k1_early_valid = false;
    // auto (k1_early 2, the default): early from 256K rows, where K1 outlasts the owned
    // masks (measured: config 3 58.7 vs ~60.5 ms); below, K1 from the count pass overlaps the
    // fill's start instead (config 2: 1.99 vs 2.07 ms)
    const bool early = ctx->k1_early == 1 || (ctx->k1_early == 2 && ctx->n >= 262144);
    if (!ctx->k1_async || !early || ctx->n < 2) return PCG_OK;
    if (!ctx->k1_stream) PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->k1_stream, cudaStreamNonBlocking));
    if (!ctx->k1_fork) PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&ctx->k1_fork, cudaEventDisableTiming));
    if (!ctx->k1_done) PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&ctx->k1_done, cudaEventDisableTiming));
    unsigned long long *anti = ctx->scal.as<unsigned long long>() + 7;
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(anti, 0, 8, s));
    PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->k1_fork, s));
    cudaStream_t ks = ctx->k1_stream;
    PCG_TRY_CUDA(ctx, cudaStreamWaitEvent(ks, ctx->k1_fork, 0));
    if (ctx->prof) cudaEventRecord(ctx->ev[0], ks);
    int64_t pairs = 0;
    int l = 0;
    int rc = run_k1(ctx, ctx->k1_shard, ctx->k1_nshards, &pairs, &l, ks, anti);
    if (rc) return rc;  // (counted in prep_launches)
    ctx->k1_early_pairs = pairs;
    if (ctx->prof) cudaEventRecord(ctx->ev[1], ks);
    PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->k1_done, ks));
    ctx->k1_pending = true;
    ctx->k1_early_valid = true;
    return PCG_OK;
}

// PCG_TRACE_PREP=1: device timestamps between the prep stages, printed to stderr (diagnostic)
struct PrepTrace {
    bool on = false;
    cudaEvent_t ev[12] = {};
    double host[12] = {};
    const char *name[12] = {};
    int k = 0;
    explicit PrepTrace(cudaStream_t s) : st(s) {
        const char *e = getenv("PCG_TRACE_PREP");
        on = e && e[0] == '1';
    }
    void mark(const char *what) {
        if (!on || k >= 12) return;
        if (!ev[k]) cudaEventCreate(&ev[k]);
        cudaEventRecord(ev[k], st);
        host[k] = std::chrono::duration<double, std::micro>(
                      std::chrono::steady_clock::now().time_since_epoch()).count();
        name[k++] = what;
    }
    ~PrepTrace() {
        if (!on) return;
        cudaStreamSynchronize(st);
        for (int i = 1; i < k; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ev[i - 1], ev[i]);
            fprintf(stderr, "prep %-22s device %8.1f us   host %8.1f us\n", name[i], ms * 1e3,
                    host[i] - host[i - 1]);
        }
        for (int i = 0; i < k; ++i) cudaEventDestroy(ev[i]);
    }
    cudaStream_t st;
};

// K0 on the device-resident raw inputs: vectors, relative lists, color buckets, bucket
// commute masks (K2a), four-Russians offsets.  Everything a build computes besides the count
// and fill passes; the benchmark times it as part of every step.
static int prep_device(pcg_ctx *ctx) {
    cudaStream_t s = ctx->stream;
    k1_join(ctx);
    ctx->deg_fused = false;
    const int64_t n_active = ctx->n, entries = ctx->entries, P = ctx->P;
    if (n_active == 0) return PCG_OK;
    if (ctx->prof) cudaEventRecord(ctx->ev[10], s);
    PrepTrace tr(s);
    tr.mark("start");
    int rc = encode_vectors(ctx, false);
    if (rc) return rc;
    PCG_ALLOC(ctx, ctx->lrel, (size_t)entries * 4);
    PCG_ALLOC(ctx, ctx->rowof, (size_t)entries * 4);
    launch_lists(ctx->lists64.as<int64_t>(), ctx->ragged ? ctx->loff.as<int64_t>() : nullptr,
                 n_active, ctx->L, entries, ctx->base, P, ctx->lrel.as<int32_t>(),
                 ctx->rowof.as<int32_t>(), ctx->bad.as<int32_t>() + 1, s);
    PCG_CHECK_LAUNCH(ctx);
    // (the invalid-code / invalid-color flags are read back with the bucket sizes below:
    // invalid colors are clamped to 0 until then, and the bit planes are not consumed before)

    tr.mark("encode+lists");
    // color buckets: stable radix sort of (color, entry) in row-major entry order, so each
    // bucket lists its rows ascending
    int end_bit = 1;
    while ((1LL << end_bit) < P) ++end_bit;
    PCG_ALLOC(ctx, ctx->eidx, (size_t)entries * 4);
    PCG_ALLOC(ctx, ctx->keys2, (size_t)entries * 4);
    PCG_ALLOC(ctx, ctx->vals2, (size_t)entries * 4);
    k_iota<<<(unsigned)((entries + 255) / 256), 256, 0, s>>>(ctx->eidx.as<int32_t>(), entries);
    size_t tmp = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceRadixSort::SortPairs(
                          nullptr, tmp, ctx->lrel.as<int32_t>(), ctx->keys2.as<int32_t>(),
                          ctx->eidx.as<int32_t>(), ctx->vals2.as<int32_t>(), (int)entries, 0,
                          end_bit, s));
    PCG_ALLOC(ctx, ctx->cubtmp, tmp);
    PCG_TRY_CUDA(ctx, cub::DeviceRadixSort::SortPairs(
                          ctx->cubtmp.p, tmp, ctx->lrel.as<int32_t>(), ctx->keys2.as<int32_t>(),
                          ctx->eidx.as<int32_t>(), ctx->vals2.as<int32_t>(), (int)entries, 0,
                          end_bit, s));
    tr.mark("radix sort");
    PCG_ALLOC(ctx, ctx->bstart, (size_t)(P + 1) * 4);
    launch_bucket_bounds(ctx->keys2.as<int32_t>(), ctx->vals2.as<int32_t>(), ctx->rowof.as<int32_t>(),
                         entries, P, ctx->bstart.as<int32_t>(), ctx->bad.as<int32_t>() + 1, s);
    PCG_CHECK_LAUNCH(ctx);

    // padded bucket starts and mask offsets (exclusive scans over P+1 colors)
    PCG_ALLOC(ctx, ctx->bpos, (size_t)(P + 1) * 4);
    PCG_ALLOC(ctx, ctx->maskoff, (size_t)(P + 1) * 8);
    cub::CountingInputIterator<int64_t> cidx(0);
    cub::TransformInputIterator<int32_t, PaddedSize, cub::CountingInputIterator<int64_t>> padded(
        cidx, PaddedSize{ctx->bstart.as<int32_t>(), P});
    cub::TransformInputIterator<int64_t, MaskWords, cub::CountingInputIterator<int64_t>> mwords(
        cidx, MaskWords{ctx->bstart.as<int32_t>(), P});
    size_t t1 = 0, t2 = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, t1, padded, ctx->bpos.as<int32_t>(),
                                                    P + 1, s));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, t2, mwords,
                                                    ctx->maskoff.as<int64_t>(), P + 1, s));
    PCG_ALLOC(ctx, ctx->cubtmp, std::max(t1, t2));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t1, padded,
                                                    ctx->bpos.as<int32_t>(), P + 1, s));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t2, mwords,
                                                    ctx->maskoff.as<int64_t>(), P + 1, s));
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->bad.as<int32_t>() + 2, 0, 4, s));
    k_bucket_max<<<(unsigned)std::min<int64_t>((P + 255) / 256, 4 * ctx->sms), 256, 0, s>>>(
        ctx->bstart.as<int32_t>(), P, ctx->bad.as<int32_t>() + 2);
    int32_t padded_total = 0, m_max = 0;
    int64_t mask_total = 0;
    int32_t bad[2] = {0, 0};
    unsigned char *hs = pinned_scratch(ctx);
    if (!hs) return fail(ctx, PCG_E_OOM, "pinned scratch allocation failed");
    // one pinned block: bad flags (8 B) | m_max (4) | padded total (4) | mask words (8)
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs, ctx->bad.p, 12, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs + 12, ctx->bpos.as<int32_t>() + P, 4, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs + 16, ctx->maskoff.as<int64_t>() + P, 8, cudaMemcpyDeviceToHost, s));
    tr.mark("bounds+scans+readback");
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    tr.mark("host sync");
    memcpy(bad, hs, 8);
    memcpy(&m_max, hs + 8, 4);
    memcpy(&padded_total, hs + 12, 4);
    memcpy(&mask_total, hs + 16, 8);
    if (bad[1] & 2) return fail(ctx, PCG_E_COLOR, "a list color lies outside the palette");
    if (bad[1] & 4) return fail(ctx, PCG_E_DUPLICATE, "a color list names the same color twice");
    if (bad[0]) {  // invalid 3-bit codes: exact raw-word predicate
        rc = encode_vectors(ctx, true);
        if (rc) return rc;
    }
    // K1 starts here, after the bucket sort (CUB's onesweep sort cannot share an SM with it)
    // and before the owned masks, the count and the fill, whose CTAs fill the SMs next to it
    rc = k1_launch_early(ctx, s);
    if (rc) return rc;
    // bucket masks when they fit comfortably (dense corners with huge buckets use the
    // partner-gather row kernel instead; both are exact).  Free memory is queried once per
    // context (and again only when a decision is close), not on every build.
    const size_t mask_bytes = (size_t)mask_total * 4;
    if (ctx->free_mem == 0 || mask_bytes > ctx->free_mem / 8) {
        size_t total_b = 0;
        cudaMemGetInfo(&ctx->free_mem, &total_b);
    }
    const size_t free_b = ctx->free_mem;
    ctx->masked = ctx->k2_mode >= 2 ||
                  (ctx->k2_mode == 0 && mask_bytes <= std::min<size_t>(free_b / 4, 24ull << 30));
    // ownership needs 12-bit member positions, 20-bit colors and <= 64 colors per list
    ctx->owned = ctx->masked && ctx->k2_mode != 2 && m_max <= 4096 && P < (1 << 20) - 1 &&
                 ctx->lmax <= 64 && ctx->kw <= 16;

    ctx->m_max = m_max;
    ctx->mask_words = mask_total;
    // +64 sentinel ids: the segmented fill loads whole 32-position words past a bucket's end
    PCG_ALLOC(ctx, ctx->bmemp, (size_t)(padded_total + 64) * 4);
    PCG_ALLOC(ctx, ctx->posof, (size_t)entries * 4);
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->bmemp.p, 0x7f, (size_t)(padded_total + 64) * 4, s));
    BucketArgs b = bucket_args(ctx);
    launch_bucket_layout(b, entries, s);
    PCG_CHECK_LAUNCH(ctx);
    tr.mark("memset+layout");
    if (ctx->masked) {
        PCG_ALLOC(ctx, ctx->masks, std::max<size_t>(mask_bytes, 16));
        b.masks = ctx->masks.as<uint32_t>();
        OwnArgs own{};
        if (ctx->owned) {
            OwnArgs &o = own;
            o.lrel = ctx->lrel.as<int32_t>();
            o.loff = ctx->ragged ? ctx->loff.as<int64_t>() : nullptr;
            o.L = ctx->L;
            o.overflow = ctx->bad.as<int32_t>() + 3;
            // table for the expected (c', k) entries of the largest bucket at load <= 1/2
            int64_t want = (int64_t)m_max * std::max(1, ctx->lmax - 1);
            int hs = 1024;
            while (hs < want && hs < 32768) hs <<= 1;
            o.hash_slots = hs;
            o.m_cap = m_max;
            o.row_lo = (int32_t)std::max<int64_t>(0, std::min(ctx->own_lo, n_active));
            o.row_hi = (int32_t)(ctx->own_hi < 0 ? n_active : std::min(ctx->own_hi, n_active));
            o.fr = ctx->own_algo == 0 ? 1 : 0;
            o.l_magic = (uint32_t)(((1ull << 32) + (uint64_t)std::max(1, ctx->L) - 1) /
                                   (uint64_t)std::max(1, ctx->L));
            if ((int64_t)m_max * std::max(1, ctx->L) >= (1 << 20)) o.fr = 0;  // umulhi range
            // direct-mapped ownership when the color table fits shared memory next to the
            // rest (16-bit member tags, two per word), rectangular lists, and groups of
            // members sharing a smaller color stay small (one level per member)
            o.dtab_words = (int32_t)(((P + 1) / 2 + 3) & ~3LL);
            o.l16 = P < 65536 ? 1 : 0;
            o.direct = (o.fr && ctx->own_direct != 0 && !ctx->ragged && P <= 28672 &&
                        (int64_t)m_max * std::max(1, ctx->lmax - 1) <= 4 * P) ? 1 : 0;
            // an exact bitmap over the colors replaces the hash table when it is smaller
            // (config 3: 15.6 + 6 KB instead of 40 KB), so that two owned-mask CTAs fit next
            // to K1 on an SM; see owned_bitmap_words
            o.bm_words = (int32_t)((((int64_t)P + 31) / 32 + 3) & ~3LL);
            // ... and while the holders of repeated colors stay well inside the holder list:
            // near the top of the palette a color's m·(L-1) items repeat ~(m(L-1))^2 / 2P
            // colors; past ~1K holders the pairing (quadratic in them) and the overflow
            // fallback cost more than the hash table (500k ids, P' = 20%, alpha = 4.5: 193 vs
            // 113 ms; config 3 sits at ~525)
            const double own_items = (double)m_max * (double)std::max(1, ctx->lmax - 1);
            o.bitmap = (o.fr && !o.direct && !ctx->ragged && ctx->own_bitmap != 0 &&
                        own_items * own_items <= 1024.0 * (double)P &&
                        owned_bitmap_words(o) < (int64_t)o.hash_slots + owned_hash_coll()) ? 1 : 0;
            // measured: staging the lists pays when they are u16 (small palettes); u32 lists
            // next to the hash table cost occupancy (config 3)
            o.stage_lists = (!ctx->ragged && o.l16) ? 1 : 0;
            // direct mode: loser lists sized for the expected number of members per color
            // that share a smaller color with an earlier member, ~ (m (L-1) / 2)^2 / P, x2
            // headroom (500k ids, P = 25000, L = 26: ~2.3k, beyond the default 1024)
            {
                const double half = (double)m_max * std::max(1, ctx->lmax - 1) / 2.0;
                const double est = half * half / (double)std::max<int64_t>(P, 1);
                int64_t lc = 1024;
                while (lc < 2.0 * est && lc < 8192) lc <<= 1;
                o.lcap = (int32_t)lc;
            }
            // shared memory: big buckets x long lists (e.g. 500k ids, P' = 2.5%, alpha = 3:
            // ~1.7k members x 39 colors) do not fit with staged lists; the direct table reads
            // the staged lists, so it goes too; if even the hash table does not fit, the
            // bucket masks without ownership (dedupe in the row passes) take over
            const size_t smem_cap = 227u * 1024u;
            if (owned_masks_smem(o, ctx->kw) > smem_cap) {
                o.stage_lists = 0;
                o.direct = 0;
            }
            if (owned_masks_smem(o, ctx->kw) > smem_cap) ctx->owned = false;
        }
        if (ctx->owned) {
            OwnArgs &o = own;
            PCG_TRY_CUDA(ctx, cudaMemsetAsync(o.overflow, 0, 4, s));
            if (ctx->dyn_work) {  // colors from an atomic counter (see work_first)
                PCG_ALLOC(ctx, ctx->workctr, 64);
                PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->workctr.p, 0, 8, s));
                o.work = ctx->workctr.as<unsigned long long>();
            }
            // the four-Russians kernel also produces the degrees (no separate K2c pass)
            const bool fr_kernel = o.fr && (ctx->kw == 2 || ctx->kw == 4 || ctx->kw == 6 || ctx->kw == 8);
            if (ctx->fuse_deg && fr_kernel) {
                PCG_ALLOC(ctx, ctx->deg, (size_t)n_active * 4);
                PCG_ALLOC(ctx, ctx->degu, (size_t)n_active * 4);
                PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->deg.p, 0, (size_t)n_active * 4, s));
                PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->degu.p, 0, (size_t)n_active * 4, s));
                o.deg = ctx->deg.as<int32_t>();
                o.degu = ctx->degu.as<int32_t>();
                ctx->deg_fused = true;
            }
            launch_owned_masks(b, o, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
            // the per-pair mask kernel (own_algo 1) always writes every row
            ctx->prep_lo = o.fr ? o.row_lo : 0;
            ctx->prep_hi = o.fr ? o.row_hi : n_active;
            ctx->own_check = true;  // the overflow flag is read back with the count totals
        }
        if (!ctx->owned) {
            launch_bucket_masks(b, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
        }
    }

    tr.mark("masks (K2a)");
    tr.mark("(end)");
    PCG_ALLOC(ctx, ctx->deg, (size_t)n_active * 4);
    PCG_ALLOC(ctx, ctx->degu, (size_t)n_active * 4);
    ctx->prep_launches = 6 + (bad[0] ? 1 : 0) + (ctx->masked ? 1 : 0) +
                         (ctx->k1_early_valid ? 1 : 0);  // + the early K1 sweep
    if (ctx->prof) {
        cudaEventRecord(ctx->ev[11], s);
        ctx->prep_timed = true;  // elapsed time read at the next host sync (count pass)
    }
    return PCG_OK;
}

extern "C" int pcg_set_inputs(pcg_ctx *ctx, const uint64_t *words, int64_t n_total,
                              int32_t nwords, int32_t num_qubits, const int64_t *active,
                              int64_t n_active, const int64_t *list_data,
                              const int64_t *list_off, int32_t list_len, int64_t palette_base,
                              int64_t palette_size) {
    if (!ctx) return PCG_E_ARG;
    ctx->err.clear();
    if (ctx->k1_pending && ctx->k1_done) cudaEventSynchronize(ctx->k1_done);  // planes reused
    ctx->k1_pending = false;
    ctx->k1_early_valid = false;
    ctx->staged = false;
    ctx->counted = false;
    if (n_active < 0 || n_total < 0 || n_active > n_total || num_qubits < 1 || nwords < 1 ||
        (int64_t)nwords * 64 < 3LL * num_qubits || palette_size < 0 || n_active > (1LL << 30))
        return fail(ctx, PCG_E_ARG, "bad build dimensions");
    if (n_active > 0 && (!words || !active || !list_data))
        return fail(ctx, PCG_E_ARG, "null input pointer");
    if (!list_off && list_len < 1 && n_active > 0)
        return fail(ctx, PCG_E_ARG, "rectangular lists need list_len >= 1");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;

    ctx->n_total = n_total;
    ctx->n = n_active;
    ctx->nwords = nwords;
    ctx->q = num_qubits;
    ctx->base = palette_base;
    // the reference's mask has ceil(P/64) (at least 1) words: every relative color below
    // that many bits is a legal list entry (driver.py:152-172)
    ctx->P = std::max<int64_t>(1, (palette_size + 63) / 64) * 64;
    palette_size = ctx->P;
    ctx->ragged = list_off != nullptr;
    ctx->npad = round_up(n_active, K1_NPAD);
    int64_t entries = 0;
    int32_t lmax = list_len;
    if (ctx->ragged) {
        entries = list_off[n_active] - list_off[0];
        lmax = 0;
        for (int64_t i = 0; i < n_active; ++i)
            lmax = std::max<int32_t>(lmax, (int32_t)(list_off[i + 1] - list_off[i]));
        if (list_off[0] != 0) return fail(ctx, PCG_E_ARG, "list_off[0] must be 0");
    } else {
        entries = n_active * (int64_t)list_len;
    }
    ctx->L = list_len;
    ctx->lmax = std::max<int32_t>(lmax, 1);
    ctx->entries = entries;
    if (entries >= (1LL << 31)) return fail(ctx, PCG_E_ARG, "too many list entries");

    PCG_ALLOC(ctx, ctx->bad, 16);
    PCG_ALLOC(ctx, ctx->scal, 64);
    if (n_active == 0) {
        ctx->kw = 2;
        ctx->staged = true;
        return PCG_OK;
    }
    PCG_ALLOC(ctx, ctx->words, (size_t)n_total * nwords * 8);
    PCG_ALLOC(ctx, ctx->active, (size_t)n_active * 8);
    PCG_ALLOC(ctx, ctx->lists64, (size_t)entries * 8);
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->words.p, words, (size_t)n_total * nwords * 8,
                                      cudaMemcpyHostToDevice, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->active.p, active, (size_t)n_active * 8,
                                      cudaMemcpyHostToDevice, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->lists64.p, list_data, (size_t)entries * 8,
                                      cudaMemcpyHostToDevice, s));
    if (ctx->ragged) {
        PCG_ALLOC(ctx, ctx->loff, (size_t)(n_active + 1) * 8);
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->loff.p, list_off, (size_t)(n_active + 1) * 8,
                                          cudaMemcpyHostToDevice, s));
    }
    ctx->staged = true;
    const int rc = prep_device(ctx);
    if (rc) ctx->staged = false;
    else ctx->launch_total += ctx->prep_launches;
    return rc;
}

// --------------------------------------------------------------------------------------
// count pass
// --------------------------------------------------------------------------------------
// 1 direct tiles, 5 four-Russians 8-bit slices (the default where supported: kw 2/4/6/8,
// q <= 128; the 4-, 5- and 6-bit four-Russians kernels were measured slower and removed)
static int k1_algo(const pcg_ctx *ctx) {
    if (ctx->k1_algo == 1) return 1;
    return fr8_supported(ctx->kw) ? 5 : 1;
}

// rows per K1 work item (measured at 1M x 64q: 2048 32.2 ms, 4096 31.1, 8192 30.1)
static int64_t fr_ichunk(const pcg_ctx *ctx) { return ctx->fr_ichunk > 0 ? ctx->fr_ichunk : 8192; }

// pairs (i<j, both < n) inside four-Russians item (jb, rows [i0,i1))
static int64_t fr_item_pairs(int64_t n, int64_t jb, int64_t i0, int64_t i1, int64_t JB) {
    const int64_t jlo = jb * JB, jhi = std::min(n, jlo + JB);
    if (jhi <= jlo) return 0;  // a padding block past the last row
    int64_t p = 0;
    const int64_t full_hi = std::min(i1, jlo);
    if (full_hi > i0) p += (full_hi - i0) * (jhi - jlo);
    const int64_t a = std::max(i0, jlo), b = std::min(i1, jhi);
    for (int64_t i = a; i < b; ++i) p += jhi - 1 - i;
    return p;
}

// pairs inside direct tiles [t0,t1) (row-major upper triangle of T x T tiles)
static int64_t direct_pairs(int64_t n, int64_t T, int64_t t0, int64_t t1) {
    int64_t p = 0, t = 0;
    for (int64_t bi = 0; bi < T && t < t1; ++bi) {
        const int64_t row_tiles = T - bi;
        const int64_t a = std::max(t0, t), b = std::min(t1, t + row_tiles);
        const int64_t rlo = bi * K1_TILE, rhi = std::min(n, rlo + (int64_t)K1_TILE);
        const int64_t rows = std::max<int64_t>(0, rhi - rlo);
        for (int64_t tt = a; tt < b; ++tt) {
            const int64_t bj = bi + (tt - t);
            const int64_t clo = bj * K1_TILE, chi = std::min(n, clo + (int64_t)K1_TILE);
            const int64_t cols = std::max<int64_t>(0, chi - clo);
            p += bi == bj ? rows * (rows - 1) / 2 : rows * cols;
        }
        t += row_tiles;
    }
    return p;
}

static int run_k1(pcg_ctx *ctx, int32_t shard, int32_t nshards, int64_t *pairs, int *launches,
                  cudaStream_t s, unsigned long long *anti) {
    const int64_t n = ctx->n;
    if (k1_algo(ctx) == 5) {
        const int64_t JB = fr8_jb(ctx->kw);
        const int64_t njb = ctx->npad / JB, ic = fr_ichunk(ctx);
        // item_start runs over the blocks in visit order; the kernel folds the triangle
        // (blocks 0, njb-1, 1, njb-2, ...) so that every CTA's item range spans about the
        // same number of table rebuilds (a short early block is paired with a long late one)
        auto jb_of = [&](int64_t v) { return fr8_fold(v, njb); };
        std::vector<int64_t> start(njb + 1, 0);
        for (int64_t v = 0; v < njb; ++v) {
            // (a padding block past the last row has no pairs and no items)
            const int64_t jlast = jb_of(v) * JB < n ? std::min(n, (jb_of(v) + 1) * JB) : 0;
            start[v + 1] = start[v] + (jlast + ic - 1) / ic;
        }
        const int64_t items = start[njb];
        const int64_t i0 = items * shard / nshards, i1 = items * (shard + 1) / nshards;
        if (nshards == 1) {
            *pairs = n * (n - 1) / 2;
        } else {
            int64_t p = 0, v = 0;
            for (int64_t it = i0; it < i1; ++it) {
                while (start[v + 1] <= it) ++v;
                const int64_t jb = jb_of(v);
                const int64_t jlast = std::min(n, (jb + 1) * JB);
                const int64_t r0 = (it - start[v]) * ic, r1 = std::min(r0 + ic, jlast);
                p += fr_item_pairs(n, jb, r0, r1, JB);
            }
            *pairs = p;
        }
        // pageable H2D: the copy is complete (staged) before cudaMemcpyAsync returns
        PCG_ALLOC(ctx, ctx->items, (size_t)(njb + 1) * 8);
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->items.p, start.data(), (size_t)(njb + 1) * 8,
                                          cudaMemcpyHostToDevice, s));
        // 8 warps when K1 shares the SMs with the row passes (its side stream), else 16
        const int warps = ctx->k1_warps > 0 ? ctx->k1_warps
                                            : (ctx->k1_stream && s == ctx->k1_stream) ? 8 : 16;
        *launches += launch_commute_fr8_items(ctx->A.as<uint32_t>(), ctx->B.as<uint32_t>(),
                                              ctx->kw, n, ctx->items.as<int64_t>(), njb,
                                              (int32_t)ic, i0, i1, anti, ctx->sms, warps, s);
    } else {
        const int64_t T = ctx->npad / K1_TILE, NT = tri_tiles(T);
        const int64_t t0 = NT * shard / nshards, t1 = NT * (shard + 1) / nshards;
        *pairs = nshards == 1 ? n * (n - 1) / 2 : direct_pairs(n, T, t0, t1);
        *launches += launch_commute_direct(ctx->A.as<uint32_t>(), ctx->B.as<uint32_t>(), ctx->kw,
                                           ctx->npad, t0, t1, anti, ctx->sms, s);
    }
    PCG_CHECK_LAUNCH(ctx);
    return PCG_OK;
}

static int32_t pick_window(const pcg_ctx *ctx) {
    if (ctx->window > 0) return (int32_t)round_up(ctx->window, 4096);
    const int64_t w = round_up(std::max<int64_t>(ctx->n, 1), 4096);
    return (int32_t)std::min<int64_t>(w, 32768);
}

static RowArgs row_args(const pcg_ctx *ctx, int64_t r0, int64_t r1) {
    RowArgs a{};
    a.n = (int32_t)ctx->n;
    a.row_begin = r0;
    a.row_end = r1;
    a.A = ctx->A.as<uint32_t>();
    a.B = ctx->B.as<uint32_t>();
    a.kw = ctx->kw;
    a.lrel = ctx->lrel.as<int32_t>();
    a.loff = ctx->ragged ? ctx->loff.as<int64_t>() : nullptr;
    a.L = ctx->L;
    a.bstart = ctx->bstart.as<int32_t>();
    a.bmem = ctx->keys2.as<int32_t>();
    if (ctx->masked) {
        a.bpos = ctx->bpos.as<int32_t>();
        a.bmemp = ctx->bmemp.as<int32_t>();
        a.posof = ctx->posof.as<int32_t>();
        a.maskoff = ctx->maskoff.as<int64_t>();
        a.masks = ctx->masks.as<uint32_t>();
    }
    a.deg = ctx->deg.as<int32_t>();
    a.degu = ctx->degu.as<int32_t>();
    a.window = pick_window(ctx);
    a.slot_cap = ctx->lmax;
    return a;
}

static int count_impl(pcg_ctx *ctx, int32_t shard, int32_t nshards, int64_t r0, int64_t r1,
                      pcg_counts *out, int *launches) {
    if (!ctx->staged) return fail(ctx, PCG_E_STATE, "pcg_count before pcg_set_inputs");
    if (nshards < 1 || shard < 0 || shard >= nshards || r0 < 0 || r1 < r0 || r1 > ctx->n)
        return fail(ctx, PCG_E_ARG, "bad shard or row range");
    if (ctx->owned && r1 > r0 && (r0 < ctx->prep_lo || r1 > ctx->prep_hi))
        return fail(ctx, PCG_E_STATE, "count rows outside the owned-mask rows of the prep "
                                      "(options own_rows_lo/own_rows_hi)");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    // an early K1 of this build (launched by the prep, own counter) is taken over by a
    // one-shard count; any other pending K1 is joined first
    const bool take_early = ctx->k1_early_valid && ctx->k1_async && shard == ctx->k1_shard &&
                            nshards == ctx->k1_nshards;
    if (!take_early) {
        k1_join(ctx);
        if (ctx->k1_early_valid) {  // a sharded count: the early sweep is not used
            ctx->k1_early_valid = false;
        }
    }
    pcg_counts c{};
    c.n_active = ctx->n;
    c.raw_words_mode = ctx->raw ? 1 : 0;
    ctx->counted = false;
    if (ctx->n < 2) {  // no pairs: every degree is zero
        if (ctx->n == 1) {
            PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->deg.p, 0, 4, s));
            PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->degu.p, 0, 4, s));
            PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
        }
        ctx->cnt_row_begin = r0;
        ctx->cnt_row_end = r1;
        ctx->last = c;
        ctx->counted = true;
        if (out) *out = c;
        return PCG_OK;
    }
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->scal.p, 0, 40, s));
    int64_t pairs = 0;
    int rc;
    // K1 only produces view_edges_scanned: with k1_async it runs on a side stream next to the
    // conflict-row passes and its count is collected later (pcg_k1_result)
    const bool async = ctx->k1_async != 0;
    cudaStream_t ks = s;
    if (async && !take_early) {
        if (!ctx->k1_stream) PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->k1_stream, cudaStreamNonBlocking));
        if (!ctx->k1_fork) PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&ctx->k1_fork, cudaEventDisableTiming));
        if (!ctx->k1_done) PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&ctx->k1_done, cudaEventDisableTiming));
        ks = ctx->k1_stream;
        PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->k1_fork, s));
        PCG_TRY_CUDA(ctx, cudaStreamWaitEvent(ks, ctx->k1_fork, 0));
    }
    if (take_early) {
        pairs = ctx->k1_early_pairs;  // this shard's pairs, already being swept
        ctx->k1_slot = 7;
    } else {
        if (ctx->prof) cudaEventRecord(ctx->ev[0], ks);
        rc = run_k1(ctx, shard, nshards, &pairs, launches, ks, ctx->scal.as<unsigned long long>());
        if (rc) return rc;
        if (ctx->prof) cudaEventRecord(ctx->ev[1], ks);
        ctx->k1_slot = 0;
        if (async) {
            PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->k1_done, ks));
            ctx->k1_pending = true;
        }
    }
    if (ctx->prof) cudaEventRecord(ctx->ev[8], s);
    const RowArgs a = row_args(ctx, r0, r1);
    if (!(ctx->owned && ctx->deg_fused))  // (fused: the prep's owned-mask kernel counted)
        *launches += ctx->owned ? launch_count_owned(a, ctx->sms, s)
                                : launch_rows(a, false, false, ctx->sms, s);
    PCG_CHECK_LAUNCH(ctx);
    if (ctx->prof) cudaEventRecord(ctx->ev[2], s);
    if (r1 > r0) {
        k_sum_degrees<<<std::min<int64_t>((r1 - r0 + 255) / 256, 4 * ctx->sms), 256, 0, s>>>(
            ctx->deg.as<int32_t>(), ctx->degu.as<int32_t>(), r0, r1,
            ctx->scal.as<unsigned long long>());
        *launches += 1;
        PCG_CHECK_LAUNCH(ctx);
    }
    unsigned long long h[5];
    int32_t ovf = 0;
    unsigned char *hs = pinned_scratch(ctx);
    if (!hs) return fail(ctx, PCG_E_OOM, "pinned scratch allocation failed");
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs + 64, ctx->scal.p, 40, cudaMemcpyDeviceToHost, s));
    if (ctx->own_check)
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs + 104, ctx->bad.as<int32_t>() + 3, 4,
                                          cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    memcpy(h, hs + 64, 40);
    if (ctx->own_check) memcpy(&ovf, hs + 104, 4);
    if (ctx->prof) {
        if (ctx->prep_timed) cudaEventElapsedTime(&ctx->ktimes[4], ctx->ev[10], ctx->ev[11]);
        ctx->prep_timed = false;
        if (!async) cudaEventElapsedTime(&ctx->ktimes[0], ctx->ev[0], ctx->ev[1]);
        cudaEventElapsedTime(&ctx->ktimes[1], ctx->ev[8], ctx->ev[2]);
    }
    if (ctx->own_check) {
        ctx->own_check = false;
        if (ovf && ctx->owned && getenv("PICASSO_DEBUG"))
            fprintf(stderr, "[picasso] ownership overflow (flag %d): bucket-mask fallback\n", ovf);
        if (ovf && ctx->owned) {  // a color's ownership table overflowed: plain bucket masks
            ctx->owned = false;   // (pairs deduplicated by the row bitmap) and count again
            BucketArgs b = bucket_args(ctx);
            launch_bucket_masks(b, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
            return count_impl(ctx, shard, nshards, r0, r1, out, launches);
        }
    }
    c.anticommuting = async ? -1 : (int64_t)h[0];  // -1: pending, see pcg_k1_result
    c.pairs_in_shard = pairs;
    c.deg_sum = (int64_t)h[1];
    c.deg_upper_sum = (int64_t)h[2];
    c.members_in_range = (int64_t)h[3];
    ctx->maxdeg = (int32_t)h[4];
    ctx->cnt_row_begin = r0;
    ctx->cnt_row_end = r1;
    ctx->last = c;
    ctx->counted = true;
    if (out) *out = c;
    return PCG_OK;
}

extern "C" int pcg_count(pcg_ctx *ctx, int32_t shard, int32_t nshards, int64_t row_begin,
                         int64_t row_end, pcg_counts *out) {
    if (!ctx) return PCG_E_ARG;
    int launches = 0;
    const int rc = count_impl(ctx, shard, nshards, row_begin, row_end, out, &launches);
    ctx->launch_total += launches;
    return rc;
}

extern "C" int pcg_copy_degrees(pcg_ctx *ctx, int32_t *deg, int32_t *deg_upper) {
    if (!ctx) return PCG_E_ARG;
    if (!ctx->counted) return fail(ctx, PCG_E_STATE, "pcg_copy_degrees before pcg_count");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    const int64_t r0 = ctx->cnt_row_begin, r1 = ctx->cnt_row_end;
    if (r1 == r0) return PCG_OK;
    cudaStream_t s = ctx->stream;
    if (deg)
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(deg, ctx->deg.as<int32_t>() + r0, (r1 - r0) * 4,
                                          cudaMemcpyDeviceToHost, s));
    if (deg_upper)
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(deg_upper, ctx->degu.as<int32_t>() + r0, (r1 - r0) * 4,
                                          cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    return PCG_OK;
}

// --------------------------------------------------------------------------------------
// fill pass
// --------------------------------------------------------------------------------------
// compact ids + row offsets from a full degree array (device pointer `deg`, n entries).
static int prefix_structures(pcg_ctx *ctx, const int32_t *deg, int64_t *n_members) {
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    PCG_ALLOC(ctx, ctx->compact, (size_t)(n + 1) * 4);
    PCG_ALLOC(ctx, ctx->rowoff, (size_t)(n + 1) * 8);
    cub::CountingInputIterator<int64_t> idx(0);
    cub::TransformInputIterator<int32_t, DegPositive, cub::CountingInputIterator<int64_t>> pos(
        idx, DegPositive{deg, n});
    cub::TransformInputIterator<int64_t, DegAt, cub::CountingInputIterator<int64_t>> dv(
        idx, DegAt{deg, n});
    size_t t1 = 0, t2 = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, t1, pos, ctx->compact.as<int32_t>(),
                                                    n + 1, s));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, t2, dv, ctx->rowoff.as<int64_t>(),
                                                    n + 1, s));
    PCG_ALLOC(ctx, ctx->cubtmp, std::max(t1, t2));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t1, pos,
                                                    ctx->compact.as<int32_t>(), n + 1, s));
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t2, dv,
                                                    ctx->rowoff.as<int64_t>(), n + 1, s));
    if (!n_members) return PCG_OK;  // caller knows the member count (no host round trip)
    int32_t nm = 0;
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&nm, ctx->compact.as<int32_t>() + n, 4,
                                      cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    *n_members = nm;
    return PCG_OK;
}



// Device -> pageable host copy of a large result: double-buffered pinned staging chunks, the
// DMA of chunk k overlapping the (OpenMP-parallel) host copy of chunk k-1.  A plain
// cudaMemcpy into pageable memory runs at a fraction of PCIe bandwidth.
static int d2h_pipelined(pcg_ctx *ctx, void *dst, const void *src, size_t bytes) {
    cudaStream_t s = ctx->stream;
    const size_t CH = 32ull << 20;
    if (bytes <= CH) {
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
        PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
        return PCG_OK;
    }
    for (int k = 0; k < 2; ++k)
        if (!ctx->stage[k]) PCG_TRY_CUDA(ctx, cudaHostAlloc(&ctx->stage[k], CH, cudaHostAllocDefault));
    const size_t nch = (bytes + CH - 1) / CH;
    auto issue = [&](size_t k) -> cudaError_t {
        const size_t off = k * CH, len = std::min(CH, bytes - off);
        cudaError_t e = cudaMemcpyAsync(ctx->stage[k & 1], static_cast<const char *>(src) + off,
                                        len, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaEventRecord(ctx->ev[6 + (k & 1)], s);
        return e;
    };
    auto drain = [&](size_t k) -> cudaError_t {
        cudaError_t e = cudaEventSynchronize(ctx->ev[6 + (k & 1)]);
        if (e != cudaSuccess) return e;
        const size_t off = k * CH, len = std::min(CH, bytes - off);
        const char *from = static_cast<const char *>(ctx->stage[k & 1]);
        char *to = static_cast<char *>(dst) + off;
        const int parts = 16;
#pragma omp parallel for num_threads(std::min(16, omp_get_num_procs())) schedule(static)
        for (int t = 0; t < parts; ++t) {
            const size_t a = len * t / parts, b = len * (t + 1) / parts;
            std::memcpy(to + a, from + a, b - a);
        }
        return cudaSuccess;
    };
    PCG_TRY_CUDA(ctx, issue(0));
    for (size_t k = 1; k < nch; ++k) {
        PCG_TRY_CUDA(ctx, issue(k));
        PCG_TRY_CUDA(ctx, drain(k - 1));
    }
    PCG_TRY_CUDA(ctx, drain(nch - 1));
    return PCG_OK;
}

// int32 -> int64 widening of one host range.  AVX-512 with non-temporal stores when the CPU
// has it: the destination is written once and never read back here, so streaming stores
// skip the read-for-ownership of every output line (1/3 less host memory traffic).
__attribute__((target("avx512f"))) static void widen_avx512(int64_t *to, const int32_t *from,
                                                              size_t len) {
    size_t x = 0;
    for (; x < len && (reinterpret_cast<uintptr_t>(to + x) & 63); ++x) to[x] = from[x];
    for (; x + 16 <= len; x += 16) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(from + x));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(from + x + 8));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(to + x), _mm512_cvtepi32_epi64(a));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(to + x + 8), _mm512_cvtepi32_epi64(b));
    }
    for (; x < len; ++x) to[x] = from[x];
    _mm_sfence();
}

static void widen_range(int64_t *to, const int32_t *from, size_t len) {
    static const bool avx512 = __builtin_cpu_supports("avx512f");
    if (avx512) {
        widen_avx512(to, from, len);
        return;
    }
    for (size_t x = 0; x < len; ++x) to[x] = from[x];
}

// In-place widening of one chunk: its int32 ids were copied into the upper half of the
// chunk's own int64 range.  Ascending order never overwrites an unread id (element x's
// int64 store ends at byte 8x+8 <= 4*len + 4x + 4, where the unread ids start), and each
// 16-id step loads before it stores.
__attribute__((target("avx512f"))) static void widen_inplace_avx512(int64_t *to, size_t len) {
    const int32_t *from = reinterpret_cast<const int32_t *>(to + len) - len;
    size_t x = 0;
    for (; x < len && (reinterpret_cast<uintptr_t>(to + x) & 63); ++x) to[x] = from[x];
    for (; x + 16 <= len; x += 16) {
        const __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(from + x));
        const __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(from + x + 8));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(to + x), _mm512_cvtepi32_epi64(a));
        _mm512_stream_si512(reinterpret_cast<__m512i *>(to + x + 8), _mm512_cvtepi32_epi64(b));
    }
    for (; x < len; ++x) to[x] = from[x];
    _mm_sfence();
}

static void widen_inplace(int64_t *to, size_t len) {
    static const bool avx512 = __builtin_cpu_supports("avx512f");
    if (avx512) {
        widen_inplace_avx512(to, len);
        return;
    }
    const int32_t *from = reinterpret_cast<const int32_t *>(to + len) - len;
    for (size_t x = 0; x < len; ++x) {
        const int64_t v = from[x];
        to[x] = v;
    }
}

// ---- byte-delta copy-out (delta.cu): decoder -------------------------------------------
// Decodes entries [x0, x1) (a whole number of rows) from their gap bytes `g` (g[0] is entry
// x0) into dst (int64, the API's output).  `rs` = the host offsets array (row starts),
// `r0` = the row of x0, `xv` = exceptions (row-major), `xc` = the exception cursor at x0.
// SIMD path: aligned 16-entry groups with no escape byte and no row start are an in-register
// prefix sum added to the running value, widened and stored with streaming stores.
template <typename G>
__attribute__((target("avx512f"))) static void delta_decode_avx512(
    int64_t *dst, const G *g, int64_t x0, int64_t x1, const int64_t *rs, int64_t r0,
    const int32_t *xv, int64_t xc) {
    constexpr uint32_t ESC = sizeof(G) == 1 ? 255u : 65535u;
    int64_t r = r0;
    int64_t next = rs[r0 + 1];  // first entry of the next row
    int32_t acc = -1;
    int64_t x = x0;
    const __m512i zero = _mm512_setzero_si512();
    while (x < x1) {
        const bool aligned = (reinterpret_cast<uintptr_t>(dst + x) & 63) == 0 && x + 16 <= x1 &&
                             next >= x + 16;
        if (aligned) {
            __m512i t;
            bool clean;
            if constexpr (sizeof(G) == 1) {
                const __m128i v = _mm_loadu_si128(reinterpret_cast<const __m128i *>(g + (x - x0)));
                clean = _mm_movemask_epi8(_mm_cmpeq_epi8(v, _mm_set1_epi8((char)255))) == 0;
                t = _mm512_cvtepu8_epi32(v);
            } else {
                const __m256i v = _mm256_loadu_si256(reinterpret_cast<const __m256i *>(g + (x - x0)));
                clean = _mm256_movemask_epi8(_mm256_cmpeq_epi16(v, _mm256_set1_epi16((short)-1))) == 0;
                t = _mm512_cvtepu16_epi32(v);
            }
            if (clean) {
                t = _mm512_add_epi32(t, _mm512_alignr_epi32(t, zero, 15));
                t = _mm512_add_epi32(t, _mm512_alignr_epi32(t, zero, 14));
                t = _mm512_add_epi32(t, _mm512_alignr_epi32(t, zero, 12));
                t = _mm512_add_epi32(t, _mm512_alignr_epi32(t, zero, 8));
                t = _mm512_add_epi32(t, _mm512_set1_epi32(acc));
                _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + x),
                                    _mm512_cvtepi32_epi64(_mm512_castsi512_si256(t)));
                _mm512_stream_si512(reinterpret_cast<__m512i *>(dst + x + 8),
                                    _mm512_cvtepi32_epi64(_mm512_extracti64x4_epi64(t, 1)));
                acc = _mm_extract_epi32(_mm512_extracti32x4_epi32(t, 3), 3);
                x += 16;
                continue;
            }
        }
        // scalar step (row starts, escapes, unaligned heads and tails)
        if (x == next) {
            ++r;
            next = rs[r + 1];
            acc = -1;
        }
        const uint32_t b = g[x - x0];
        acc = b == ESC ? xv[xc++] : acc + (int32_t)b;
        dst[x] = acc;
        ++x;
    }
    _mm_sfence();
}

template <typename G>
static void delta_decode_scalar(int64_t *dst, const G *g, int64_t x0, int64_t x1,
                                const int64_t *rs, int64_t r0, const int32_t *xv, int64_t xc) {
    constexpr uint32_t ESC = sizeof(G) == 1 ? 255u : 65535u;
    int64_t r = r0, next = rs[r0 + 1];
    int32_t acc = -1;
    for (int64_t x = x0; x < x1; ++x) {
        if (x == next) {
            ++r;
            next = rs[r + 1];
            acc = -1;
        }
        const uint32_t b = g[x - x0];
        acc = b == ESC ? xv[xc++] : acc + (int32_t)b;
        dst[x] = acc;
    }
}

template <typename G>
static void delta_decode(bool simd, int64_t *dst, const void *g, int64_t x0, int64_t x1,
                         const int64_t *rs, int64_t r0, const int32_t *xv, int64_t xc) {
    const G *gg = static_cast<const G *>(g);
    if (simd) delta_decode_avx512<G>(dst, gg, x0, x1, rs, r0, xv, xc);
    else delta_decode_scalar<G>(dst, gg, x0, x1, rs, r0, xv, xc);
}

// Public-build copy-out of the neighbor ids: byte-delta encode on the device, copy gap bytes
// (pipelined per worker, row-aligned chunks) + exceptions, decode on the host into `dst`.
// `offsets` is the host copy of the CSR offsets (nm+1 entries, already transferred).
static int d2h_delta(pcg_ctx *ctx, int64_t *dst, const int64_t *offsets, int64_t nm, int64_t nnz) {
    cudaStream_t s = ctx->stream;
    // gap width: bytes while the mean gap (ids per row / entries per row) is small
    const double mean_gap = nnz > 0 ? (double)ctx->n * (double)nm / (double)nnz : 0.0;
    const bool wide = ctx->d2h_gap16 == 1 || (ctx->d2h_gap16 == 0 && mean_gap > 64.0);
    const size_t gb = wide ? 2 : 1;  // bytes per gap
    PCG_ALLOC(ctx, ctx->dbytes, (size_t)nnz * gb);
    PCG_ALLOC(ctx, ctx->dxcnt, (size_t)(nm + 1) * 4);
    PCG_ALLOC(ctx, ctx->dxoff, (size_t)(nm + 1) * 8);
    launch_delta(false, wide, ctx->nbr_o.as<int32_t>(), ctx->offsets_o.as<int64_t>(), nm,
                 ctx->dbytes.p, ctx->dxcnt.as<int32_t>(), nullptr, nullptr, ctx->sms, s);
    PCG_CHECK_LAUNCH(ctx);
    cub::CountingInputIterator<int64_t> idx(0);
    cub::TransformInputIterator<int64_t, DegAt, cub::CountingInputIterator<int64_t>> xc(
        idx, DegAt{ctx->dxcnt.as<int32_t>(), nm});
    size_t tmp = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, xc, ctx->dxoff.as<int64_t>(), nm + 1, s));
    PCG_ALLOC(ctx, ctx->cubtmp, tmp);
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, tmp, xc, ctx->dxoff.as<int64_t>(), nm + 1, s));
    if (ctx->hxoff_cap < (size_t)(nm + 1)) {
        if (ctx->hxoff) cudaFreeHost(ctx->hxoff);
        ctx->hxoff = nullptr;
        PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&ctx->hxoff), (size_t)(nm + 1) * 8, cudaHostAllocDefault));
        ctx->hxoff_cap = (size_t)(nm + 1);
    }
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->hxoff, ctx->dxoff.p, (size_t)(nm + 1) * 8, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    const int64_t X = ctx->hxoff[nm];
    PCG_ALLOC(ctx, ctx->dxval, (size_t)std::max<int64_t>(X, 1) * 4);
    launch_delta(true, wide, ctx->nbr_o.as<int32_t>(), ctx->offsets_o.as<int64_t>(), nm, nullptr,
                 nullptr, ctx->dxoff.as<int64_t>(), ctx->dxval.as<int32_t>(), ctx->sms, s);
    PCG_CHECK_LAUNCH(ctx);
    if (ctx->hx_cap < (size_t)std::max<int64_t>(X, 1)) {
        if (ctx->hxval) cudaFreeHost(ctx->hxval);
        ctx->hxval = nullptr;
        ctx->hx_cap = (size_t)std::max<int64_t>(X, 1) + ((size_t)std::max<int64_t>(X, 1) >> 2);
        PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&ctx->hxval), ctx->hx_cap * 4, cudaHostAllocDefault));
    }
    if (X > 0)
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->hxval, ctx->dxval.p, (size_t)X * 4, cudaMemcpyDeviceToHost, s));
    ctx->copy_bytes += (int64_t)nnz * (int64_t)gb + X * 4 + (nm + 1) * 8;  // gaps, exceptions, offsets
    // row-aligned chunks of ~CH entries
    const int64_t CH = ctx->d2h_chunk > 0 ? ctx->d2h_chunk : (int64_t)1 << 19;
    std::vector<int64_t> cr;  // chunk row bounds
    cr.push_back(0);
    while (cr.back() < nm) {
        const int64_t want = offsets[cr.back()] + CH;
        int64_t r = std::upper_bound(offsets + cr.back() + 1, offsets + nm + 1, want) - offsets - 1;
        if (r <= cr.back()) r = cr.back() + 1;  // a row longer than CH: its own chunk
        cr.push_back(std::min<int64_t>(r, nm));
    }
    const size_t nch = cr.size() - 1;
    size_t maxb = 0;
    for (size_t k = 0; k < nch; ++k)
        maxb = std::max<size_t>(maxb, (size_t)(offsets[cr[k + 1]] - offsets[cr[k]]) * gb);
    const int W = ctx->d2h_threads > 0 ? ctx->d2h_threads : std::min(16, omp_get_num_procs());
    if (ctx->hbytes_cap < maxb || (int)ctx->hbytes.size() < 2 * W) {
        for (uint8_t *p : ctx->hbytes)
            if (p) cudaFreeHost(p);
        ctx->hbytes.assign(2 * W, nullptr);
        ctx->hbytes_cap = std::max<size_t>(maxb, (size_t)CH * gb);
        for (int k = 0; k < 2 * W; ++k)
            PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&ctx->hbytes[k]), ctx->hbytes_cap, cudaHostAllocDefault));
    }
    while ((int)ctx->ring_ev.size() < 2 * W + 1) {
        cudaEvent_t e;
        PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ring_ev.push_back(e);
    }
    while ((int)ctx->ring_st.size() < W) {
        cudaStream_t st;
        PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ctx->ring_st.push_back(st);
    }
    cudaEvent_t ready = ctx->ring_ev[2 * W];
    PCG_TRY_CUDA(ctx, cudaEventRecord(ready, s));  // bytes + exceptions queued before it
    static const bool simd = __builtin_cpu_supports("avx512f");
    const uint8_t *src = ctx->dbytes.as<uint8_t>();  // gap array, gb bytes per entry
    int failed = 0;
#pragma omp parallel num_threads(W)
    {
        const int w = omp_get_thread_num();
        cudaSetDevice(ctx->device);
        cudaStream_t st = ctx->ring_st[w];
        cudaStreamWaitEvent(st, ready, 0);
        auto issue = [&](size_t k, int slot) -> cudaError_t {
            const int64_t b0 = offsets[cr[k]], b1 = offsets[cr[k + 1]];
            cudaError_t e = cudaMemcpyAsync(ctx->hbytes[2 * w + slot], src + b0 * gb,
                                            (size_t)(b1 - b0) * gb, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ring_ev[2 * w + slot], st);
            return e;
        };
        const size_t Wt = (size_t)omp_get_num_threads();  // the team may be smaller than W
        int slot = 0;
        if ((size_t)w < nch && issue(w, 0) != cudaSuccess) failed = 1;
        if (cudaEventSynchronize(ready) != cudaSuccess) failed = 1;  // exceptions on the host
        for (size_t k = w; k < nch && !failed; k += Wt, slot ^= 1) {
            if (k + Wt < nch && issue(k + Wt, slot ^ 1) != cudaSuccess) failed = 1;
            if (cudaEventSynchronize(ctx->ring_ev[2 * w + slot]) != cudaSuccess) {
                failed = 1;
                break;
            }
            const int64_t r0 = cr[k], x0 = offsets[r0], x1 = offsets[cr[k + 1]];
            if (wide)
                delta_decode<uint16_t>(simd, dst, ctx->hbytes[2 * w + slot], x0, x1, offsets, r0,
                                       ctx->hxval, ctx->hxoff[r0]);
            else
                delta_decode<uint8_t>(simd, dst, ctx->hbytes[2 * w + slot], x0, x1, offsets, r0,
                                      ctx->hxval, ctx->hxoff[r0]);
        }
        cudaStreamSynchronize(st);
    }
    if (failed) return fail(ctx, PCG_E_CUDA, "delta copy-out failed");
    return PCG_OK;
}

static int fill_rows_device(pcg_ctx *ctx, int64_t r0, int64_t r1, const int32_t *deg,
                            int32_t maxdeg, bool identity, void *out, int64_t out_base,
                            int *launches, bool out64 = true, const int32_t *rows_list = nullptr);

// Public build, pipelined: the member rows are cut into pieces (whole copy-out chunks).  For
// each piece the build stream runs the fill (rows via the member -> row list), the gap count,
// a piece-local scan of the exception counts, a small readback of the piece's exception
// offsets (their total sizes the exception copy), the gap/exception write and the exception
// D2H; host workers decode the chunks of every finished piece while later pieces are filled.
static int fill_delta_pipe(pcg_ctx *ctx, int64_t *dst, const int64_t *offsets, int64_t nm,
                           int64_t nnz, int *launches, bool pinned_dst) {
    cudaStream_t s = ctx->stream;
    const double mean_gap = nnz > 0 ? (double)ctx->n * (double)nm / (double)nnz : 0.0;
    const bool wide = ctx->d2h_gap16 == 1 || (ctx->d2h_gap16 == 0 && mean_gap > 64.0);
    const size_t gb = wide ? 2 : 1;
    PCG_ALLOC(ctx, ctx->dbytes, (size_t)nnz * gb);
    PCG_ALLOC(ctx, ctx->dxcnt, (size_t)(nm + 1) * 4);
    PCG_ALLOC(ctx, ctx->dxoff, (size_t)(nm + 1) * 8);
    if (ctx->hxoff_cap < (size_t)(nm + 1)) {
        if (ctx->hxoff) cudaFreeHost(ctx->hxoff);
        ctx->hxoff = nullptr;
        PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&ctx->hxoff), (size_t)(nm + 1) * 8, cudaHostAllocDefault));
        ctx->hxoff_cap = (size_t)(nm + 1);
    }
    // copy-out chunks (row-aligned, ~CH entries) and pieces (runs of whole chunks)
    const int64_t CH = ctx->d2h_chunk > 0 ? ctx->d2h_chunk : (int64_t)1 << 19;
    std::vector<int64_t> cr;
    cr.push_back(0);
    while (cr.back() < nm) {
        const int64_t want = offsets[cr.back()] + CH;
        int64_t r = std::upper_bound(offsets + cr.back() + 1, offsets + nm + 1, want) - offsets - 1;
        if (r <= cr.back()) r = cr.back() + 1;
        cr.push_back(std::min<int64_t>(r, nm));
    }
    const int64_t nch = (int64_t)cr.size() - 1;
    // measured at c2 (16 host cores): 8-12 pieces with 15 decoders best (e2e median 14.3-14.5
    // ms vs 16.3-18.9 for fill-then-copy-out); 24 pieces lose to the per-piece readbacks
    const int64_t want_pieces = ctx->d2h_pieces > 0 ? ctx->d2h_pieces : 8;
    const int64_t cpp = std::max<int64_t>(1, (nch + want_pieces - 1) / want_pieces);  // chunks per piece
    const int64_t K = (nch + cpp - 1) / cpp;
    // chunks shipped as int64 by DMA straight into a pinned destination (evenly spread), the
    // rest as gaps decoded by the host: the copy engine and the decoders share the host
    // memory bandwidth
    const int dma_pct = pinned_dst ? (ctx->d2h_dma >= 0 ? std::min(ctx->d2h_dma, 100) : 0) : 0;
    std::vector<char> direct(nch, 0);
    std::vector<int64_t> dmaoff(nch, 0);
    std::vector<int64_t> todo;  // the decoders' chunks
    int64_t dma_entries = 0;
    for (int64_t k = 0; k < nch; ++k) {
        direct[k] = ((k + 1) * dma_pct / 100) > (k * dma_pct / 100);
        if (direct[k]) {
            dmaoff[k] = dma_entries;
            dma_entries += offsets[cr[k + 1]] - offsets[cr[k]];
        } else {
            todo.push_back(k);
        }
    }
    if (dma_entries > 0) {
        PCG_ALLOC(ctx, ctx->dwide, (size_t)dma_entries * 8);
        if (!ctx->dma_st) PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->dma_st, cudaStreamNonBlocking));
    }
    const int64_t ntodo = (int64_t)todo.size();
    size_t maxb = 0;
    for (int64_t k = 0; k < nch; ++k)
        maxb = std::max<size_t>(maxb, (size_t)(offsets[cr[k + 1]] - offsets[cr[k]]) * gb);
    // decoders: one core is left to the orchestrating thread
    const int W = ctx->d2h_threads > 0 ? ctx->d2h_threads
                                       : std::max(1, std::min(16, omp_get_num_procs() - 1));
    if (ctx->hbytes_cap < maxb || (int)ctx->hbytes.size() < 2 * W) {
        for (uint8_t *p : ctx->hbytes)
            if (p) cudaFreeHost(p);
        ctx->hbytes.assign(2 * W, nullptr);
        ctx->hbytes_cap = std::max<size_t>(maxb, (size_t)CH * gb);
        for (int k = 0; k < 2 * W; ++k)
            PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&ctx->hbytes[k]), ctx->hbytes_cap, cudaHostAllocDefault));
    }
    while ((int)ctx->ring_ev.size() < 2 * W + 1) {
        cudaEvent_t e;
        PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ring_ev.push_back(e);
    }
    while ((int)ctx->ring_st.size() < W) {
        cudaStream_t st;
        PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ctx->ring_st.push_back(st);
    }
    while ((int64_t)ctx->piece_ev.size() < K) {  // blocking-sync: waiters sleep, not spin
        cudaEvent_t e;
        PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming | cudaEventBlockingSync));
        ctx->piece_ev.push_back(e);
    }
    if (!ctx->scan_ev) PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&ctx->scan_ev, cudaEventDisableTiming | cudaEventBlockingSync));
    while ((int64_t)ctx->hxpiece.size() < K) ctx->hxpiece.push_back({nullptr, 0});
    // the scan's temporary storage, sized for the largest piece
    cub::CountingInputIterator<int64_t> idx(0);
    size_t tmp = 0;
    {
        cub::TransformInputIterator<int64_t, DegAt, cub::CountingInputIterator<int64_t>> xc(
            idx, DegAt{ctx->dxcnt.as<int32_t>(), nm});
        PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, xc, ctx->dxoff.as<int64_t>(), nm + 1, s));
    }
    PCG_ALLOC(ctx, ctx->cubtmp, tmp);
    // device exceptions of one piece (row starts + long gaps); grown inside a piece if needed
    PCG_ALLOC(ctx, ctx->dxval, (size_t)(2 * (nm + nnz / 16) / K + 1024) * 4);
    static const bool simd = __builtin_cpu_supports("avx512f");
    const uint8_t *src = ctx->dbytes.as<uint8_t>();
    std::atomic<int64_t> ready(0);  // pieces whose exceptions are queued for the host
    std::atomic<int> failed(0);
    int orc = PCG_OK;
    int64_t xbytes = 0;

    // one piece on the build stream; returns a status (runs on the orchestrating thread)
    auto run_piece = [&](int64_t p) -> int {
        const int64_t m0 = cr[p * cpp], m1 = cr[std::min(nch, (p + 1) * cpp)];
        int rc = fill_rows_device(ctx, m0, m1, ctx->deg.as<int32_t>(), ctx->maxdeg, nm == ctx->n,
                                  ctx->nbr_o.p, 0, launches, /*out64=*/false, ctx->mrow.as<int32_t>());
        if (rc) return rc;
        const int64_t rows = m1 - m0;
        launch_delta(false, wide, ctx->nbr_o.as<int32_t>(), ctx->offsets_o.as<int64_t>() + m0, rows,
                     ctx->dbytes.p, ctx->dxcnt.as<int32_t>() + m0, nullptr, nullptr, ctx->sms, s);
        PCG_CHECK_LAUNCH(ctx);
        cub::TransformInputIterator<int64_t, DegAt, cub::CountingInputIterator<int64_t>> xc(
            idx, DegAt{ctx->dxcnt.as<int32_t>() + m0, rows});
        size_t t = tmp;
        PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t, xc, ctx->dxoff.as<int64_t>() + m0, rows + 1, s));
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->hxoff + m0, ctx->dxoff.as<int64_t>() + m0, (size_t)(rows + 1) * 8,
                                          cudaMemcpyDeviceToHost, s));
        PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->scan_ev, s));
        PCG_TRY_CUDA(ctx, cudaEventSynchronize(ctx->scan_ev));
        const int64_t X = ctx->hxoff[m1];  // exceptions of this piece (piece-relative offsets)
        auto &hp = ctx->hxpiece[p];
        if (hp.second < (size_t)std::max<int64_t>(X, 1)) {
            if (hp.first) cudaFreeHost(hp.first);
            hp.first = nullptr;
            hp.second = (size_t)std::max<int64_t>(X, 1) + ((size_t)std::max<int64_t>(X, 1) >> 2);
            PCG_TRY_CUDA(ctx, cudaHostAlloc(reinterpret_cast<void **>(&hp.first), hp.second * 4, cudaHostAllocDefault));
        }
        PCG_ALLOC(ctx, ctx->dxval, (size_t)std::max<int64_t>(X, 1) * 4);
        launch_delta(true, wide, ctx->nbr_o.as<int32_t>(), ctx->offsets_o.as<int64_t>() + m0, rows, nullptr,
                     nullptr, ctx->dxoff.as<int64_t>() + m0, ctx->dxval.as<int32_t>(), ctx->sms, s);
        PCG_CHECK_LAUNCH(ctx);
        if (X > 0)
            PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hp.first, ctx->dxval.p, (size_t)X * 4, cudaMemcpyDeviceToHost, s));
        bool any_direct = false;
        for (int64_t k = p * cpp; k < std::min(nch, (p + 1) * cpp); ++k) {
            if (!direct[k]) continue;
            const int64_t x0 = offsets[cr[k]], x1 = offsets[cr[k + 1]];
            *launches += launch_widen(ctx->nbr_o.as<int32_t>() + x0, ctx->dwide.as<int64_t>() + dmaoff[k],
                                      x1 - x0, ctx->sms, s);
            any_direct = true;
        }
        PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->piece_ev[p], s));
        if (any_direct) {
            PCG_TRY_CUDA(ctx, cudaStreamWaitEvent(ctx->dma_st, ctx->piece_ev[p], 0));
            for (int64_t k = p * cpp; k < std::min(nch, (p + 1) * cpp); ++k) {
                if (!direct[k]) continue;
                const int64_t x0 = offsets[cr[k]], x1 = offsets[cr[k + 1]];
                PCG_TRY_CUDA(ctx, cudaMemcpyAsync(dst + x0, ctx->dwide.as<int64_t>() + dmaoff[k],
                                                  (size_t)(x1 - x0) * 8, cudaMemcpyDeviceToHost, ctx->dma_st));
            }
        }
        xbytes += X * 4 + (rows + 1) * 8;
        return PCG_OK;
    };

    // orchestrator: pieces in order on the build stream (its own thread, so it exists whatever
    // team size OpenMP grants the decoders)
    std::thread orch([&] {
        cudaSetDevice(ctx->device);
        for (int64_t p = 0; p < K && !failed.load(); ++p) {
            const int rc = run_piece(p);
            if (rc) {
                orc = rc;
                failed.store(1);
            }
            ready.store(p + 1, std::memory_order_release);
        }
        ready.store(K, std::memory_order_release);
    });
#pragma omp parallel num_threads(W)
    {
        const int w = omp_get_thread_num();
        const int Wt = omp_get_num_threads();  // the team may be smaller than W
        cudaSetDevice(ctx->device);
        {  // decoder w: chunks w, w+Wt, ... double-buffered on its own stream
            cudaStream_t st = ctx->ring_st[w];
            auto piece_ready = [&](int64_t k) { return ready.load(std::memory_order_acquire) > k / cpp; };
            auto issue = [&](int64_t k, int slot) -> cudaError_t {
                cudaError_t e = cudaStreamWaitEvent(st, ctx->piece_ev[k / cpp], 0);
                const int64_t b0 = offsets[cr[k]], b1 = offsets[cr[k + 1]];
                if (e == cudaSuccess)
                    e = cudaMemcpyAsync(ctx->hbytes[2 * w + slot], src + b0 * gb, (size_t)(b1 - b0) * gb,
                                        cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaEventRecord(ctx->ring_ev[2 * w + slot], st);
                return e;
            };
            int64_t issued = w - Wt;  // last of the decoders' chunks (index into todo) queued
            int slot = 0;
            for (int64_t j = w; j < ntodo && !failed.load(); j += Wt, slot ^= 1) {
                const int64_t k = todo[j];
                if (issued < j) {  // not prefetched: wait for its piece, then copy it
                    while (!piece_ready(k) && !failed.load())  // sleep: leave the core to the
                        std::this_thread::sleep_for(std::chrono::microseconds(10));  // orchestrator
                    if (failed.load() || issue(k, slot) != cudaSuccess) {
                        failed.store(1);
                        break;
                    }
                    issued = j;
                }
                // prefetch the next chunk only if its piece is already out (never wait here)
                if (j + Wt < ntodo && piece_ready(todo[j + Wt])) {
                    if (issue(todo[j + Wt], slot ^ 1) != cudaSuccess) {
                        failed.store(1);
                        break;
                    }
                    issued = j + Wt;
                }
                const int64_t p = k / cpp;
                // the piece's exceptions and offsets are on the host once its event completed
                if (cudaEventSynchronize(ctx->piece_ev[p]) != cudaSuccess ||
                    cudaEventSynchronize(ctx->ring_ev[2 * w + slot]) != cudaSuccess) {
                    failed.store(1);
                    break;
                }
                const int64_t r0 = cr[k], x0 = offsets[r0], x1 = offsets[cr[k + 1]];
                const int32_t *xv = ctx->hxpiece[p].first;
                if (wide)
                    delta_decode<uint16_t>(simd, dst, ctx->hbytes[2 * w + slot], x0, x1, offsets, r0, xv, ctx->hxoff[r0]);
                else
                    delta_decode<uint8_t>(simd, dst, ctx->hbytes[2 * w + slot], x0, x1, offsets, r0, xv, ctx->hxoff[r0]);
            }
            cudaStreamSynchronize(st);
        }
    }
    orch.join();
    if (dma_entries > 0 && cudaStreamSynchronize(ctx->dma_st) != cudaSuccess) failed.store(1);
    if (orc) return orc;
    if (failed.load()) return fail(ctx, PCG_E_CUDA, "pipelined fill / delta copy-out failed");
    // gaps of the decoded chunks, int64 of the DMA chunks, exceptions and their offsets
    ctx->copy_bytes += (nnz - dma_entries) * (int64_t)gb + dma_entries * 8 + xbytes;
    return PCG_OK;
}

// D2H straight into a pinned (registered) int64 destination: every chunk's int32 ids land in
// the upper half of its own int64 range and are widened there by the worker that owns the
// chunk — no staging buffer, so host DRAM sees the DMA writes and the int64 stores only.
static int d2h_widen_direct(pcg_ctx *ctx, int64_t *dst, const int32_t *src, size_t count) {
    const size_t CH = ctx->d2h_chunk > 0 ? (size_t)ctx->d2h_chunk : (size_t)1 << 20;  // ids
    const int W = ctx->d2h_threads > 0 ? ctx->d2h_threads : std::min(16, omp_get_num_procs());
    const size_t nch = (count + CH - 1) / CH;
    if (nch == 0) return PCG_OK;
    while (ctx->chunk_ev.size() < nch) {
        cudaEvent_t e;
        PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->chunk_ev.push_back(e);
    }
    // all copies queued up front on the build stream (after the fill), in chunk order
    for (size_t k = 0; k < nch; ++k) {
        const size_t off = k * CH, len = std::min(CH, count - off);
        int32_t *half = reinterpret_cast<int32_t *>(dst + off + len) - len;
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(half, src + off, len * 4, cudaMemcpyDeviceToHost, ctx->stream));
        PCG_TRY_CUDA(ctx, cudaEventRecord(ctx->chunk_ev[k], ctx->stream));
    }
    int failed = 0;
#pragma omp parallel for num_threads(W) schedule(static, 1)
    for (long k = 0; k < (long)nch; ++k) {
        if (cudaEventSynchronize(ctx->chunk_ev[k]) != cudaSuccess) {
            failed = 1;
            continue;
        }
        const size_t off = (size_t)k * CH, len = std::min(CH, count - off);
        widen_inplace(dst + off, len);
    }
    if (failed) return fail(ctx, PCG_E_CUDA, "direct D2H copy failed");
    return PCG_OK;
}

// Same pipeline, int32 device ids widened to the API's int64 during the host-side copy, so
// only half the bytes cross PCIe.  W host workers (one OpenMP region for the whole copy), each
// with its own stream and two pinned staging chunks: worker w takes chunks w, w+W, ...; it
// keeps the DMA of its next chunk in flight while it widens the current one, so the copy
// engines and all host cores stay busy without a per-chunk fork/join.  (The e2e at config 2
// is bound by host memory traffic: 0.83 GB of DMA writes and 1.66 GB of int64 stores.)
static int d2h_widen(pcg_ctx *ctx, int64_t *dst, const int32_t *src, size_t count) {
    const size_t CH = ctx->d2h_chunk > 0 ? (size_t)ctx->d2h_chunk : (size_t)1 << 20;  // ids
    const int W = ctx->d2h_threads > 0 ? ctx->d2h_threads : std::min(16, omp_get_num_procs());
    const size_t nch = (count + CH - 1) / CH;
    if (nch == 0) return PCG_OK;
    if (ctx->ring_bytes != CH * 4 || (int)ctx->ring.size() != 2 * W) {
        for (void *p : ctx->ring)
            if (p) cudaFreeHost(p);
        ctx->ring.assign(2 * W, nullptr);
        ctx->ring_bytes = CH * 4;
        for (int k = 0; k < 2 * W; ++k)
            PCG_TRY_CUDA(ctx, cudaHostAlloc(&ctx->ring[k], CH * 4, cudaHostAllocDefault));
    }
    while ((int)ctx->ring_ev.size() < 2 * W + 1) {
        cudaEvent_t e;
        PCG_TRY_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->ring_ev.push_back(e);
    }
    while ((int)ctx->ring_st.size() < W) {
        cudaStream_t st;
        PCG_TRY_CUDA(ctx, cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ctx->ring_st.push_back(st);
    }
    // the workers' streams start after everything queued on the build stream (the fill)
    cudaEvent_t ready = ctx->ring_ev[2 * W];
    PCG_TRY_CUDA(ctx, cudaEventRecord(ready, ctx->stream));
    int failed = 0;
#pragma omp parallel num_threads(W)
    {
        const int w = omp_get_thread_num();
        cudaSetDevice(ctx->device);
        cudaStream_t st = ctx->ring_st[w];
        cudaStreamWaitEvent(st, ready, 0);
        auto issue = [&](size_t k, int slot) -> cudaError_t {
            const size_t off = k * CH, len = std::min(CH, count - off);
            if (ctx->d2h_mode == 2) return cudaEventRecord(ctx->ring_ev[2 * w + slot], st);  // widen only
            cudaError_t e = cudaMemcpyAsync(ctx->ring[2 * w + slot], src + off, len * 4,
                                            cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->ring_ev[2 * w + slot], st);
            return e;
        };
        const size_t Wt = (size_t)omp_get_num_threads();  // the team may be smaller than W
        int slot = 0;
        if ((size_t)w < nch && issue(w, 0) != cudaSuccess) failed = 1;
        for (size_t k = w; k < nch && !failed; k += Wt, slot ^= 1) {
            if (k + Wt < nch && issue(k + Wt, slot ^ 1) != cudaSuccess) failed = 1;
            if (cudaEventSynchronize(ctx->ring_ev[2 * w + slot]) != cudaSuccess) {
                failed = 1;
                break;
            }
            const size_t off = k * CH, len = std::min(CH, count - off);
            if (ctx->d2h_mode != 1)  // (diagnostic mode 1: copies only)
                widen_range(dst + off, static_cast<const int32_t *>(ctx->ring[2 * w + slot]), len);
        }
        cudaStreamSynchronize(st);
    }
    if (failed) return fail(ctx, PCG_E_CUDA, "pipelined D2H copy failed");
    return PCG_OK;
}

// Fill pass for rows [r0, r1) into `out` (int64, entry index out_base at out[0]).  Owned
// masks: the bins fill (sparse rows, > 128K ids), the block fill (<= 128K ids) or the
// segmented fill (dense rows); lists longer than 64 colors and the non-owned mask modes take
// the lane-per-bucket bitmap row kernel.
static int fill_rows_device(pcg_ctx *ctx, int64_t r0, int64_t r1, const int32_t *deg,
                            int32_t maxdeg, bool identity, void *out, int64_t out_base,
                            int *launches, bool out64, const int32_t *rows_list) {
    cudaStream_t s = ctx->stream;
    RowArgs a = row_args(ctx, r0, r1);
    if (rows_list) a.rows_list = rows_list;  // [r0, r1) index this list of rows
    a.deg = const_cast<int32_t *>(deg);
    a.rowoff = ctx->rowoff.as<int64_t>();
    a.compact = identity ? nullptr : ctx->compact.as<int32_t>();
    a.out = out;
    a.out_base = out_base;
    if (!ctx->owned) {
        *launches += launch_rows(a, true, out64, ctx->sms, s);
        PCG_CHECK_LAUNCH(ctx);
        return PCG_OK;
    }
    // the bins fill (counting sort per row, bins sorted by bitonic networks) is the default
    // from 40K ids when the longest row fits its list.  Measured (block fill vs bins): 20K ids
    // 0.204 vs 0.230 ms, 50K 0.611 vs 0.587, 100K (config 2) 1.368 vs 1.256, 140K 2.33 vs
    // 2.02; 1M (config 3) 20.7 ms vs the segmented fill's 52.8
    const bool bins_auto = ctx->fill_algo == 0 && ctx->n >= 40000;
    // measured (500k ids): rows up to 16K ids still win with the bins fill (P' = 20%,
    // alpha = 4.5, mean row 8.5k: 36.9 ms with 384 threads vs the segmented fill's 52.9)
    const int32_t bins_maxdeg = ctx->bins_maxdeg > 0 ? ctx->bins_maxdeg : 16384;
    if ((ctx->fill_algo == 7 || bins_auto) && ctx->mask_words < (1LL << 32) && maxdeg <= bins_maxdeg) {
        // bins fill (sparse rows): counting sort of each row's admitted ids
        BinArgs g{};
        const double mean = ctx->n > 0 ? (double)ctx->last.deg_sum / (double)ctx->n : 1.0;
        bins_geometry(ctx->n, mean, ctx->bins_threads, &g);
        if (ctx->bins_shift != 0) {  // testing/tuning: bin width 2^(auto + delta)
            g.shift = std::max(0, std::min(30, g.shift + ctx->bins_shift));
            g.nbins = (int32_t)((std::max<int64_t>(ctx->n, 1) + (1LL << g.shift) - 1) >> g.shift);
        }
        const int wpm = (ctx->m_max + 31) / 32;
        g.lcap = (ctx->lmax + 3) & ~3;
        g.dcap = (int)std::min<int64_t>(4096, ((int64_t)ctx->lmax * wpm + 7) & ~7);
        if (ctx->blk_dcap > 0) g.dcap = (ctx->blk_dcap + 7) & ~7;
        g.ecap = (std::max(maxdeg, 1) + 31) & ~31;
        if (bins_smem_bytes(g) <= 227u * 1024u && g.nbins <= (1 << 16)) {
            RowArgs ab = a;
            if (ctx->dyn_work) {  // rows from an atomic counter (see work_first)
                PCG_ALLOC(ctx, ctx->workctr, 64);
                PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->workctr.as<unsigned long long>() + 1, 0, 8, s));
                ab.work = ctx->workctr.as<unsigned long long>() + 1;
            }
            *launches += launch_fill_bins(ab, g, out64, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
            return PCG_OK;
        }
    }
    // measured (c2, 100k ids): block fill 1.37-1.40 ms vs segmented 1.68 ms; at 1M ids the
    // segmented fill's narrower windows win, so the block fill is the default up to 128K ids
    const bool blk_auto = ctx->fill_algo == 0 && ctx->n <= 131072;  // (and bins did not fit)
    if ((ctx->fill_algo == 5 || blk_auto) && ctx->mask_words < (1LL << 32)) {
        // block fill: one CTA per row, bitmap over the whole id range (or wide windows)
        BlkArgs g{};
        blk_geometry(ctx->n, ctx->blk_threads, ctx->blk_groups, &g);
        const int wpm = (ctx->m_max + 31) / 32;
        g.lcap = (ctx->lmax + 3) & ~3;
        g.dcap = (int)std::min<int64_t>(4096, ((int64_t)ctx->lmax * (wpm + (g.nwin > 1 ? 1 : 0)) + 7) & ~7);
        if (ctx->blk_dcap > 0) g.dcap = (ctx->blk_dcap + 7) & ~7;  // testing: chunked descriptors
        // admitted-id list: sized for a window of the longest row (+ slack for uneven windows);
        // a window that overflows it re-decodes its descriptors instead
        // the row's list holds a window of the longest row (+25% when windows split rows
        // unevenly); a window that overflows it re-decodes its descriptors instead
        const int64_t per_win = (int64_t)maxdeg / g.nwin + (g.nwin > 1 ? maxdeg / (4 * g.nwin) : 0);
        g.ecap = (int32_t)std::min<int64_t>(16384, (per_win + 31) & ~31);
        if (ctx->blk_ecap != 0) g.ecap = ctx->blk_ecap < 0 ? 0 : (ctx->blk_ecap + 7) & ~7;
        if (blk_smem_bytes(g, g.groups) <= 227u * 1024u) {
            if (g.nwin > 1) {
                PCG_ALLOC(ctx, ctx->bnd, (size_t)ctx->P * (g.nwin + 1) * 4);
                *launches += launch_window_bounds(ctx->bstart.as<int32_t>(), ctx->bpos.as<int32_t>(),
                                                  ctx->bmemp.as<int32_t>(), ctx->P, g.nwin, g.wb,
                                                  ctx->bnd.as<int32_t>(), s);
                g.bnd = ctx->bnd.as<int32_t>();
            }
            *launches += launch_fill_blk(a, g, out64, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
            return PCG_OK;
        }
    }
    if ((ctx->fill_algo == 0 || ctx->fill_algo == 6) && ctx->mask_words < (1LL << 32) && ctx->lmax <= 64 &&
        maxdeg < 65535) {
        // segmented fill (default): warp-decoded mask words, lane-segment harvest
        SegArgs g{};
        // measured: small windows (more warps per SM) win at config 2; at 1M ids fewer,
        // larger windows win (each window re-decodes the words that straddle its edges)
        const int64_t max_bits = ctx->seg_bits > 0 ? ctx->seg_bits : (ctx->n <= 131072 ? 33792 : 64512);
        seg_geometry(ctx->n, max_bits, &g.wb, &g.nwin, &g.seg);
        const int wpm = (ctx->m_max + 31) / 32;
        g.desc_cap = (ctx->lmax * (wpm + (g.nwin > 1 ? 1 : 0)) + 7) & ~7;  // x8 padding
        g.warp_words = ((g.wb >> 5) + 32 + 2 * g.desc_cap + 3) & ~3;
        g.warps = ctx->seg_warps > 0 ? ctx->seg_warps : (ctx->n <= 131072 ? 2 : 4);
        if ((size_t)g.warp_words * 4 * g.warps <= 227u * 1024u) {
            if (g.nwin > 1) {
                PCG_ALLOC(ctx, ctx->bnd, (size_t)ctx->P * (g.nwin + 1) * 4);
                *launches += launch_window_bounds(ctx->bstart.as<int32_t>(), ctx->bpos.as<int32_t>(),
                                                  ctx->bmemp.as<int32_t>(), ctx->P, g.nwin, g.wb,
                                                  ctx->bnd.as<int32_t>(), s);
                g.bnd = ctx->bnd.as<int32_t>();
            }
            *launches += launch_fill_seg(a, g, out64, ctx->sms, s);
            PCG_CHECK_LAUNCH(ctx);
            return PCG_OK;
        }
    }
    // lane-per-bucket bitmap fill: lists longer than 64 colors, rows of 64K+ ids
    *launches += launch_rows(a, true, out64, ctx->sms, s);
    PCG_CHECK_LAUNCH(ctx);
    return PCG_OK;
}

static int fill_impl(pcg_ctx *ctx, bool to_host, int64_t *members, int64_t *offsets,
                     int64_t *neighbors, int *launches) {
    if (!ctx->counted || ctx->cnt_row_begin != 0 || ctx->cnt_row_end != ctx->n)
        return fail(ctx, PCG_E_STATE, "pcg_fill needs a count over all rows first");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n;
    const int64_t nm = ctx->last.members_in_range, nnz = ctx->last.deg_sum;
    if (to_host && n < 2) {
        if (offsets) offsets[0] = 0;
        return PCG_OK;
    }
    if (n < 2) return PCG_OK;
    if (ctx->prof) cudaEventRecord(ctx->ev[3], s);
    // the member count is the count pass's (rows with degree > 0), no readback needed
    int rc = prefix_structures(ctx, ctx->deg.as<int32_t>(), nullptr);
    if (rc) return rc;
    PCG_ALLOC(ctx, ctx->members_o, (size_t)std::max<int64_t>(nm, 1) * 8);
    PCG_ALLOC(ctx, ctx->offsets_o, (size_t)(nm + 1) * 8);
    PCG_ALLOC(ctx, ctx->nbr_o, (size_t)std::max<int64_t>(nnz, 1) * 4);
    // public build with the delta copy-out: the fill runs in pieces inside the copy-out, each
    // piece overlapping the host decode of the previous ones
    const bool pipe = to_host && neighbors && offsets && nnz > 0 && ctx->d2h_mode == 0 && ctx->d2h_pipe != 0;
    if (pipe) PCG_ALLOC(ctx, ctx->mrow, (size_t)std::max<int64_t>(nm, 1) * 4);
    *launches += launch_compact(ctx->deg.as<int32_t>(), n,
                                nm == n ? nullptr : ctx->compact.as<int32_t>(),
                                ctx->rowoff.as<int64_t>(), ctx->active.as<int64_t>(),
                                ctx->members_o.as<int64_t>(), ctx->offsets_o.as<int64_t>(),
                                pipe ? ctx->mrow.as<int32_t>() : nullptr, s);
    PCG_CHECK_LAUNCH(ctx);
    if (ctx->prof) cudaEventRecord(ctx->ev[4], s);
    if (nnz > 0 && !pipe) {
        rc = fill_rows_device(ctx, 0, n, ctx->deg.as<int32_t>(), ctx->maxdeg, nm == n,
                              ctx->nbr_o.p, 0, launches, /*out64=*/false);
        if (rc) return rc;
    }
    if (ctx->prof) cudaEventRecord(ctx->ev[5], s);
    if (to_host) {
        ctx->copy_bytes = (nm > 0 && members ? nm * 8 : 0) + (offsets ? (nm + 1) * 8 : 0);
        if (nm > 0 && members)
            PCG_TRY_CUDA(ctx, cudaMemcpyAsync(members, ctx->members_o.p, nm * 8,
                                              cudaMemcpyDeviceToHost, s));
        if (offsets)
            PCG_TRY_CUDA(ctx, cudaMemcpyAsync(offsets, ctx->offsets_o.p, (nm + 1) * 8,
                                              cudaMemcpyDeviceToHost, s));
    }
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    if (to_host && nnz > 0 && neighbors) {
        cudaPointerAttributes at{};
        const bool pinned = cudaPointerGetAttributes(&at, neighbors) == cudaSuccess &&
                            at.type == cudaMemoryTypeHost;
        cudaGetLastError();
        if (pipe)  // pieces of fill + delta copy-out (default)
            rc = fill_delta_pipe(ctx, neighbors, offsets, nm, nnz, launches, pinned);
        else if (ctx->d2h_mode == 0 && offsets)  // delta copy-out after the whole fill
            rc = d2h_delta(ctx, neighbors, offsets, nm, nnz);
        else if (pinned && ctx->d2h_mode == 3)
            rc = d2h_widen_direct(ctx, neighbors, ctx->nbr_o.as<int32_t>(), (size_t)nnz);
        else
            rc = d2h_widen(ctx, neighbors, ctx->nbr_o.as<int32_t>(), (size_t)nnz);
        if (ctx->d2h_mode != 0 || !offsets) ctx->copy_bytes += nnz * 4;
        if (rc) return rc;
    }
    if (ctx->prof) {
        cudaEventElapsedTime(&ctx->ktimes[3], ctx->ev[3], ctx->ev[4]);
        cudaEventElapsedTime(&ctx->ktimes[2], ctx->ev[4], ctx->ev[5]);
    }
    return PCG_OK;
}

extern "C" int pcg_fill(pcg_ctx *ctx, int64_t *members, int64_t *offsets, int64_t *neighbors) {
    if (!ctx) return PCG_E_ARG;
    int launches = 0;
    const int rc = fill_impl(ctx, true, members, offsets, neighbors, &launches);
    ctx->launch_total += launches;
    return rc;
}

extern "C" int pcg_count_device(pcg_ctx *ctx, pcg_counts *out, int32_t *launches) {
    if (!ctx) return PCG_E_ARG;
    int l = 0;
    int rc = count_impl(ctx, 0, 1, 0, ctx->n, out, &l);
    ctx->launch_total += l;
    if (launches) *launches = l;
    return rc;
}

extern "C" int pcg_k1_result(pcg_ctx *ctx, int64_t *anticommuting) {
    if (!ctx || !anticommuting) return PCG_E_ARG;
    if (!ctx->counted) return fail(ctx, PCG_E_STATE, "pcg_k1_result before pcg_count");
    if (ctx->k1_pending) {
        PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
        unsigned long long a = 0;
        unsigned char *hs = pinned_scratch(ctx);
        if (!hs) return fail(ctx, PCG_E_OOM, "pinned scratch allocation failed");
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(hs + 128, ctx->scal.as<unsigned long long>() + ctx->k1_slot, 8,
                                          cudaMemcpyDeviceToHost, ctx->k1_stream));
        PCG_TRY_CUDA(ctx, cudaStreamSynchronize(ctx->k1_stream));
        memcpy(&a, hs + 128, 8);
        if (ctx->prof) cudaEventElapsedTime(&ctx->ktimes[0], ctx->ev[0], ctx->ev[1]);
        ctx->last.anticommuting = (int64_t)a;
        ctx->k1_pending = false;
    }
    *anticommuting = ctx->last.anticommuting;
    return PCG_OK;
}

extern "C" int pcg_build_device(pcg_ctx *ctx, pcg_counts *out, int32_t *launches) {
    if (!ctx) return PCG_E_ARG;
    if (!ctx->staged) return fail(ctx, PCG_E_STATE, "pcg_build_device before pcg_set_inputs");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    int rc = prep_device(ctx);
    if (rc) return rc;
    int l = ctx->prep_launches;
    rc = count_impl(ctx, 0, 1, 0, ctx->n, out, &l);
    if (rc) return rc;
    rc = fill_impl(ctx, false, nullptr, nullptr, nullptr, &l);
    ctx->launch_total += l;
    if (launches) *launches = l;
    if (rc) return rc;
    if (ctx->k1_pending) {
        int64_t anti = 0;
        rc = pcg_k1_result(ctx, &anti);
        if (rc) return rc;
        if (out) out->anticommuting = anti;
    }
    return PCG_OK;
}

extern "C" int pcg_fill_device(pcg_ctx *ctx, int32_t *launches) {
    if (!ctx) return PCG_E_ARG;
    int l = 0;
    int rc = fill_impl(ctx, false, nullptr, nullptr, nullptr, &l);
    ctx->launch_total += l;
    if (launches) *launches = l;
    return rc;
}

extern "C" int pcg_fill_rows(pcg_ctx *ctx, const int32_t *global_deg, int64_t *neighbors,
                             int64_t *slice_begin, int64_t *slice_end) {
    if (!ctx || !global_deg || !slice_begin || !slice_end) return PCG_E_ARG;
    if (!ctx->counted) return fail(ctx, PCG_E_STATE, "pcg_fill_rows before pcg_count");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n, r0 = ctx->cnt_row_begin, r1 = ctx->cnt_row_end;
    if (n < 2) {
        *slice_begin = *slice_end = 0;
        return PCG_OK;
    }
    PCG_ALLOC(ctx, ctx->gdeg, (size_t)n * 4);
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->gdeg.p, global_deg, n * 4, cudaMemcpyHostToDevice, s));
    int64_t nm = 0;
    int rc = prefix_structures(ctx, ctx->gdeg.as<int32_t>(), &nm);
    if (rc) return rc;
    int64_t lohi[2];
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&lohi[0], ctx->rowoff.as<int64_t>() + r0, 8,
                                      cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&lohi[1], ctx->rowoff.as<int64_t>() + r1, 8,
                                      cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    *slice_begin = lohi[0];
    *slice_end = lohi[1];
    if (!neighbors) return PCG_OK;
    const int64_t cnt = lohi[1] - lohi[0];
    if (cnt == 0) return PCG_OK;
    PCG_ALLOC(ctx, ctx->nbr_o, (size_t)cnt * 8);
    int32_t gmax = 0;
    for (int64_t r = r0; r < r1; ++r) gmax = std::max(gmax, global_deg[r]);
    int l = 0;
    rc = fill_rows_device(ctx, r0, r1, ctx->gdeg.as<int32_t>(), gmax, nm == n, ctx->nbr_o.p,
                          lohi[0], &l);
    ctx->launch_total += l + 3;  // + the prefix scans and compaction
    if (rc) return rc;
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    return d2h_pipelined(ctx, neighbors, ctx->nbr_o.p, (size_t)cnt * 8);
}

// Device-pointer variants for the sharded build (NCCL collectives operate on the caller's
// device tensors; nothing crosses PCIe).
extern "C" int pcg_degrees_device(pcg_ctx *ctx, int32_t *deg_dev) {
    if (!ctx || !deg_dev) return PCG_E_ARG;
    if (!ctx->counted) return fail(ctx, PCG_E_STATE, "pcg_degrees_device before pcg_count");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    const int64_t r0 = ctx->cnt_row_begin, r1 = ctx->cnt_row_end;
    if (r1 > r0)
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(deg_dev, ctx->deg.as<int32_t>() + r0, (r1 - r0) * 4,
                                          cudaMemcpyDeviceToDevice, ctx->stream));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PCG_OK;
}

extern "C" int pcg_fill_rows_device(pcg_ctx *ctx, const int32_t *global_deg_dev, int32_t maxdeg,
                                    int64_t *neighbors_dev, int64_t *slice_begin,
                                    int64_t *slice_end) {
    if (!ctx || !global_deg_dev || !slice_begin || !slice_end) return PCG_E_ARG;
    if (!ctx->counted) return fail(ctx, PCG_E_STATE, "pcg_fill_rows_device before pcg_count");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int64_t n = ctx->n, r0 = ctx->cnt_row_begin, r1 = ctx->cnt_row_end;
    if (n < 2) {
        *slice_begin = *slice_end = 0;
        return PCG_OK;
    }
    PCG_ALLOC(ctx, ctx->gdeg, (size_t)n * 4);
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->gdeg.p, global_deg_dev, n * 4,
                                      cudaMemcpyDeviceToDevice, s));
    int64_t nm = 0;
    int rc = prefix_structures(ctx, ctx->gdeg.as<int32_t>(), &nm);
    if (rc) return rc;
    int64_t lohi[2];
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&lohi[0], ctx->rowoff.as<int64_t>() + r0, 8,
                                      cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&lohi[1], ctx->rowoff.as<int64_t>() + r1, 8,
                                      cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    *slice_begin = lohi[0];
    *slice_end = lohi[1];
    if (!neighbors_dev || lohi[1] == lohi[0]) return PCG_OK;
    int l = 0;
    // option "rows_out_abs": neighbors_dev is the whole CSR's base (the rows land at their
    // global offsets: the root's exchange buffer), not the slice's.
    // option "rows_out32": the slice is written as int32 (a sharded build all-gathers half
    // the bytes and widens after the exchange)
    rc = fill_rows_device(ctx, r0, r1, ctx->gdeg.as<int32_t>(), maxdeg, nm == n, neighbors_dev,
                          ctx->rows_out_abs ? 0 : lohi[0], &l, /*out64=*/ctx->rows_out32 == 0);
    ctx->launch_total += l + 3;  // + the prefix scans and compaction
    if (rc) return rc;
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    return PCG_OK;
}

extern "C" int64_t pcg_launch_total(const pcg_ctx *ctx) { return ctx ? ctx->launch_total : 0; }

extern "C" int pcg_prep_device(pcg_ctx *ctx) {
    if (!ctx) return PCG_E_ARG;
    if (!ctx->staged) return fail(ctx, PCG_E_STATE, "pcg_prep_device before pcg_set_inputs");
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    ctx->counted = false;
    const int rc = prep_device(ctx);
    if (!rc) ctx->launch_total += ctx->prep_launches;
    return rc;
}

// Palette lists on the device (rng.py:22-70, driver.py:175-188): active ids in, (n, L) int64
// colors out (host pointers); base_key = mix64(seed + phi * iteration), computed by the caller
// exactly like rng.stream_keys.
extern "C" int pcg_assign_lists(pcg_ctx *ctx, const int64_t *active, int64_t n, uint64_t base_key,
                                int64_t palette_size, int32_t list_size, int64_t palette_base,
                                int64_t *out) {
    if (!ctx || (n > 0 && (!active || !out))) return PCG_E_ARG;
    if (list_size < 1 || list_size > 1024 || palette_size < list_size)
        return fail(ctx, PCG_E_ARG, "need 0 < list_size <= palette_size, list_size <= 1024");
    if (n == 0) return PCG_OK;
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    PCG_ALLOC(ctx, ctx->active, (size_t)n * 8);
    PCG_ALLOC(ctx, ctx->lists64, (size_t)n * list_size * 8);
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->active.p, active, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    launch_assign_lists(ctx->active.as<int64_t>(), n, base_key, palette_size, list_size, palette_base,
                        ctx->lists64.as<int64_t>(), s);
    PCG_CHECK_LAUNCH(ctx);
    int rc = d2h_pipelined(ctx, out, ctx->lists64.p, (size_t)n * list_size * 8);
    ctx->staged = false;  // the staging buffers now hold lists, not a build's inputs
    return rc;
}

// --------------------------------------------------------------------------------------
// exhaustive validator (validation.py:41-131, exhaustive mode)
// --------------------------------------------------------------------------------------
namespace {
struct CountAt {
    const int64_t *c;
    int64_t n;
    __host__ __device__ int64_t operator()(int64_t i) const { return i < n ? c[i] : 0; }
};
}  // namespace

extern "C" int pcg_validate(pcg_ctx *ctx, const uint64_t *words, int64_t n_total, int32_t nwords,
                            int32_t num_qubits, const int64_t *active, int64_t n_active,
                            const int64_t *color, int32_t cap, int64_t *pairs_out,
                            int64_t *violations, int64_t *edges) {
    if (!ctx || !violations || !edges) return PCG_E_ARG;
    ctx->err.clear();
    if (ctx->k1_pending && ctx->k1_done) cudaEventSynchronize(ctx->k1_done);
    ctx->k1_pending = false;
    ctx->k1_early_valid = false;
    ctx->staged = false;  // the validator reuses the build's staging buffers
    ctx->counted = false;
    if (n_active < 0 || n_total < 0 || n_active > n_total || num_qubits < 1 || nwords < 1 ||
        (int64_t)nwords * 64 < 3LL * num_qubits || n_active > (1LL << 30) || cap < 0)
        return fail(ctx, PCG_E_ARG, "bad validation dimensions");
    if (n_active > 0 && (!words || !active || !color)) return fail(ctx, PCG_E_ARG, "null input pointer");
    if (cap > 0 && !pairs_out) return fail(ctx, PCG_E_ARG, "null pairs_out");
    *violations = 0;
    *edges = 0;
    if (n_active < 2) return PCG_OK;
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    ctx->n_total = n_total;
    ctx->n = n_active;
    ctx->nwords = nwords;
    ctx->q = num_qubits;
    ctx->npad = round_up(n_active, K1_NPAD);
    PCG_ALLOC(ctx, ctx->bad, 16);
    PCG_ALLOC(ctx, ctx->scal, 64);
    PCG_ALLOC(ctx, ctx->words, (size_t)n_total * nwords * 8);
    PCG_ALLOC(ctx, ctx->active, (size_t)n_active * 8);
    PCG_ALLOC(ctx, ctx->vcolor, (size_t)n_active * 8);
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->words.p, words, (size_t)n_total * nwords * 8,
                                      cudaMemcpyHostToDevice, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->active.p, active, (size_t)n_active * 8,
                                      cudaMemcpyHostToDevice, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(ctx->vcolor.p, color, (size_t)n_active * 8,
                                      cudaMemcpyHostToDevice, s));
    // bit planes (raw 3-bit words when a code is invalid: the exact predicate either way)
    int rc = encode_vectors(ctx, false);
    if (rc) return rc;
    int32_t bad = 0;
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&bad, ctx->bad.p, 4, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    if (bad) {
        rc = encode_vectors(ctx, true);
        if (rc) return rc;
    }
    // |E|: the commuting-pair sweep (K1)
    PCG_TRY_CUDA(ctx, cudaMemsetAsync(ctx->scal.p, 0, 64, s));
    int64_t pairs = 0;
    int launches = 0;
    rc = run_k1(ctx, 0, 1, &pairs, &launches, s, ctx->scal.as<unsigned long long>());
    if (rc) return rc;
    // color classes: stable sort of (color, local index)
    const int64_t n = n_active;
    PCG_ALLOC(ctx, ctx->vkeys, (size_t)n * 8);
    PCG_ALLOC(ctx, ctx->vkeys2, (size_t)n * 8);
    PCG_ALLOC(ctx, ctx->vvals, (size_t)n * 4);
    PCG_ALLOC(ctx, ctx->vvals2, (size_t)n * 4);
    PCG_ALLOC(ctx, ctx->vcnt, (size_t)(n + 1) * 8);
    PCG_ALLOC(ctx, ctx->voff, (size_t)(n + 1) * 8);
    launch_class_keys(ctx->vcolor.as<int64_t>(), n, ctx->vkeys.as<int64_t>(),
                      ctx->vvals.as<int32_t>(), s);
    PCG_CHECK_LAUNCH(ctx);
    size_t tmp = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceRadixSort::SortPairs(nullptr, tmp, ctx->vkeys.as<int64_t>(),
                                                      ctx->vkeys2.as<int64_t>(), ctx->vvals.as<int32_t>(),
                                                      ctx->vvals2.as<int32_t>(), (int)n, 0, 64, s));
    PCG_ALLOC(ctx, ctx->cubtmp, tmp);
    PCG_TRY_CUDA(ctx, cub::DeviceRadixSort::SortPairs(ctx->cubtmp.p, tmp, ctx->vkeys.as<int64_t>(),
                                                      ctx->vkeys2.as<int64_t>(), ctx->vvals.as<int32_t>(),
                                                      ctx->vvals2.as<int32_t>(), (int)n, 0, 64, s));
    launch_class_pairs(false, ctx->vkeys2.as<int64_t>(), ctx->vvals2.as<int32_t>(), n,
                       ctx->A.as<uint32_t>(), ctx->B.as<uint32_t>(), ctx->kw,
                       ctx->vcnt.as<int64_t>(), nullptr, 0, nullptr, s);
    PCG_CHECK_LAUNCH(ctx);
    cub::CountingInputIterator<int64_t> idx(0);
    cub::TransformInputIterator<int64_t, CountAt, cub::CountingInputIterator<int64_t>> cv(
        idx, CountAt{ctx->vcnt.as<int64_t>(), n});
    size_t t2 = 0;
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, t2, cv, ctx->voff.as<int64_t>(), n + 1, s));
    PCG_ALLOC(ctx, ctx->cubtmp, t2);
    PCG_TRY_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->cubtmp.p, t2, cv, ctx->voff.as<int64_t>(), n + 1, s));
    int64_t total = 0;
    unsigned long long anti = 0;
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&total, ctx->voff.as<int64_t>() + n, 8, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaMemcpyAsync(&anti, ctx->scal.p, 8, cudaMemcpyDeviceToHost, s));
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    *violations = total;
    *edges = pairs - (int64_t)anti;
    const int64_t take = std::min<int64_t>(total, cap);
    if (take > 0) {
        PCG_ALLOC(ctx, ctx->vpairs, (size_t)take * 16);
        launch_class_pairs(true, ctx->vkeys2.as<int64_t>(), ctx->vvals2.as<int32_t>(), n,
                           ctx->A.as<uint32_t>(), ctx->B.as<uint32_t>(), ctx->kw, nullptr,
                           ctx->voff.as<int64_t>(), take, ctx->vpairs.as<int64_t>(), s);
        PCG_CHECK_LAUNCH(ctx);
        PCG_TRY_CUDA(ctx, cudaMemcpyAsync(pairs_out, ctx->vpairs.p, (size_t)take * 16,
                                          cudaMemcpyDeviceToHost, s));
        PCG_TRY_CUDA(ctx, cudaStreamSynchronize(s));
    }
    return PCG_OK;
}

// Pin (register) / unpin a host range for direct DMA: the reused host output buffer of the
// public build (hostpool.py) is registered once, so later builds copy straight into it.
extern "C" int pcg_host_register(void *ptr, uint64_t bytes, int32_t on) {
    if (!ptr || bytes == 0) return PCG_E_ARG;
    cudaError_t e = on ? cudaHostRegister(ptr, (size_t)bytes, cudaHostRegisterDefault)
                       : cudaHostUnregister(ptr);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return PCG_E_CUDA;
    }
    return PCG_OK;
}

// Bytes the last pcg_fill copied device -> host (members, offsets and the encoded neighbor
// ids), for the benchmark's e2e accounting.
extern "C" int64_t pcg_last_copy_bytes(const pcg_ctx *ctx) { return ctx ? ctx->copy_bytes : 0; }

// --------------------------------------------------------------------------------------
// Multi-GPU exchange through peer memory (distributed.py, exchange="p2p").  The root rank
// exports one device buffer (the canonical CSR's int32 ids); every rank maps it and its fill
// (pcg_fill_rows_device with rows_out32) stores its rows straight into the root's HBM over
// NVLink as they are produced — the slice transfer overlaps the fill row by row, with no
// separate gather.  Handles are CUDA IPC handles (64 bytes), exchanged by the caller's
// process group; a buffer is reused (and its handle stays valid) while it is large enough.
// --------------------------------------------------------------------------------------
extern "C" int pcg_exchange_buffer(pcg_ctx *ctx, uint64_t bytes, void **dptr, uint8_t *handle) {
    if (!ctx || !dptr || !handle) return PCG_E_ARG;
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    PCG_ALLOC(ctx, ctx->xbuf, (size_t)bytes);
    if (ctx->xhandle_of != ctx->xbuf.p) {
        PCG_TRY_CUDA(ctx, cudaIpcGetMemHandle(&ctx->xhandle, ctx->xbuf.p));
        ctx->xhandle_of = ctx->xbuf.p;
    }
    *dptr = ctx->xbuf.p;
    memcpy(handle, &ctx->xhandle, sizeof(cudaIpcMemHandle_t));
    return PCG_OK;
}

extern "C" int pcg_exchange_map(pcg_ctx *ctx, const uint8_t *handle, void **dptr) {
    if (!ctx || !dptr || !handle) return PCG_E_ARG;
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    const std::string key(reinterpret_cast<const char *>(handle), sizeof(cudaIpcMemHandle_t));
    for (auto &m : ctx->xmaps)
        if (m.first == key) {
            *dptr = m.second;
            return PCG_OK;
        }
    // a new buffer from this peer (it grew): drop the old mappings
    for (auto &m : ctx->xmaps) cudaIpcCloseMemHandle(m.second);
    ctx->xmaps.clear();
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *p = nullptr;
    PCG_TRY_CUDA(ctx, cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    ctx->xmaps.emplace_back(key, p);
    *dptr = p;
    return PCG_OK;
}

// int32 ids in device memory -> the int64 host array (pinned or pageable), widened on the
// way (the root's copy-out of the exchanged CSR)
extern "C" int pcg_ids_to_host(pcg_ctx *ctx, const int32_t *src_dev, int64_t count, int64_t *dst) {
    if (!ctx || count < 0 || (count > 0 && (!src_dev || !dst))) return PCG_E_ARG;
    if (count == 0) return PCG_OK;
    PCG_TRY_CUDA(ctx, cudaSetDevice(ctx->device));
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, dst) == cudaSuccess &&
                        at.type == cudaMemoryTypeHost;
    cudaGetLastError();
    const int rc = pinned ? d2h_widen_direct(ctx, dst, src_dev, (size_t)count)
                          : d2h_widen(ctx, dst, src_dev, (size_t)count);
    if (rc) return rc;
    PCG_TRY_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return PCG_OK;
}
