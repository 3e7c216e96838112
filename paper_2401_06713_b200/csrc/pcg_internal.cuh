// Internal declarations of the B200 conflict-graph builder (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/picasso_b200.h"

namespace pcg {

// Every launcher raises a kernel's dynamic shared memory cap to the most the kernel can take
// (the device's opt-in maximum minus the kernel's static shared memory: the same value from
// every thread), never to the size of its own launch: a per-launch cap races between host
// threads launching the same kernel with different sizes (one thread's smaller cap lands just
// before the other's launch: invalid argument).  The cap is not an allocation; occupancy
// follows each launch's actual request.
// L2 eviction priorities for the fills (PTX createpolicy + .L2::cache_hint): the bucket
// member gathers are kept (evict_last) while the streaming owned-mask reads and the CSR
// writes go first, so the 130 MB member array at config 3 stays mostly L2-resident.
__device__ __forceinline__ uint64_t l2_policy_keep() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_stream() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ int32_t ldg_pol(const int32_t *ptr, uint64_t pol) {
    int32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ldg_pol(const uint32_t *ptr, uint64_t pol) {
    uint32_t v;
    asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(ptr), "l"(pol));
    return v;
}
__device__ __forceinline__ void stg_pol(int32_t *ptr, int32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.s32 [%0], %1, %2;" ::"l"(ptr), "r"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void stg_pol(int64_t *ptr, int32_t v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.s64 [%0], %1, %2;" ::"l"(ptr), "l"((int64_t)v), "l"(pol)
                 : "memory");
}

template <typename F>
inline void allow_max_smem(F kern) {
    static const int optin = [] {
        int d = 0, v = 0;
        cudaGetDevice(&d);
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
        return v;
    }();
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, kern) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             optin - (int)fa.sharedSizeBytes) != cudaSuccess)
        cudaGetLastError();  // the launch itself reports a request above the cap
}

// The SM's L1/shared split is set when a CTA lands on an idle SM, from the kernel's preferred
// carveout.  K1 (136 KB of tables) would otherwise get the smallest split that fits it and
// leave no shared memory for the owned-mask and fill CTAs meant to run next to it: the
// kernels that share SMs ask for the whole carveout.
template <typename F>
inline void prefer_max_shared(F kern) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared) != cudaSuccess)
        cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Device memory: grow-only buffers owned by one context.
// ---------------------------------------------------------------------------
struct DevBuf {
    void *p = nullptr;
    size_t cap = 0;
    template <typename T>
    T *as() const { return static_cast<T *>(p); }
};

cudaError_t ensure(DevBuf &b, size_t bytes);
void release(DevBuf &b);

// ---------------------------------------------------------------------------
// Geometry of the commuting-pair sweep (K1).
// ---------------------------------------------------------------------------
constexpr int K1_TILE = 128;  // rows == cols of one upper-triangle tile (direct kernel)
constexpr int K1_NPAD = 2048;   // rows of the bit planes are padded to a multiple of this

// ---------------------------------------------------------------------------
// Arguments of the conflict-row kernels (K2).
// ---------------------------------------------------------------------------
struct RowArgs {
    int32_t n;              // active rows of the build
    int64_t row_begin, row_end;
    const uint32_t *B;      // (npad, kw) partner vectors
    const uint32_t *A;      // (npad, kw) row vectors
    int32_t kw;
    const int32_t *lrel;    // colors relative to palette_base, CSR by row
    const int64_t *loff;    // (n+1) row offsets into lrel, or null (rectangular, L each)
    int32_t L;
    const int32_t *bstart;  // (P+1) color bucket starts
    const int32_t *bmem;    // bucket members (ascending local ids per bucket)
    int32_t *deg;           // count pass: full conflict degree per row
    int32_t *degu;          // count pass: partners j > i per row
    const int64_t *rowoff;  // fill pass: (n+1) exclusive prefix of deg
    const int32_t *compact; // fill pass: compact id per local row (null = identity)
    void *out;              // fill pass: neighbor slice (int64 or int32)
    int64_t out_base;       // global entry index of out[0]
    int32_t window;         // bitmap window (bits), multiple of 4096
    int32_t slot_cap;       // color slots reserved per warp (>= max list length)
    // bucket-mask mode (K2a + K2b): no partner gathers in the row pass
    const int32_t *bpos;    // (P+1) 4-aligned start of each padded bucket in bmemp
    const int32_t *bmemp;   // padded bucket members (ascending local ids, pad = sentinel)
    const int32_t *posof;   // per list entry: position of its row inside the color's bucket
    const int64_t *maskoff; // (P+1) word offset of each color's commute-mask matrix
    const uint32_t *masks;  // per color: m rows of ceil(m/32) words, bit t = commute(k, t)
    const int32_t *rows_list; // if set: process rows rows_list[row_begin..row_end) instead
    unsigned long long *work; // if set (zeroed): rows handed out by an atomic counter
};

struct OwnArgs {
    const int32_t *lrel;   // relative colors of every list entry
    const int64_t *loff;   // ragged row offsets or null
    int32_t L;
    int32_t *overflow;     // set when a color's ownership table overflowed
    int32_t hash_slots;    // power of two
    int32_t m_cap;         // >= largest bucket
    int32_t fr;            // 1: four-Russians mask kernel (kw in {2,4,6,8})
    uint32_t l_magic;      // ceil(2^32 / L): item -> member by umulhi
    int32_t direct;        // 1: direct-mapped ownership table over the colors (small P)
    int32_t dtab_words;    // its size (>= P, multiple of 4)
    int32_t l16;           // members' lists staged as u16 (palette < 65536)
    int32_t stage_lists;   // stage the members' lists in shared memory (direct mode, or u16)
    int32_t lcap;          // direct mode: losers per level (0: 1024)
    int32_t bitmap;        // 1: an exact bitmap over the colors instead of the hash table
    int32_t bm_words;      // its words (>= P/32, multiple of 4)
    int32_t row_lo, row_hi;  // four-Russians kernel: mask rows only for members in [lo, hi)
                             // (a sharded build's own rows; other rows are left unwritten)
    unsigned long long *work;  // if set (zeroed): colors handed out by an atomic counter
    int32_t *deg, *degu;       // if set (zeroed): the four-Russians kernel also adds each
                               // mask row's popcounts (the count pass's degrees)
};

// Work distribution of the persistent row/color loops.  Static (item += gridDim.x) when
// `work` is null; otherwise every CTA takes the next item from an atomic counter, so the
// CTAs that are resident take all the work — the ones that only fit once the concurrently
// running K1 has drained find the counter exhausted.  Block-uniform; `slot` is __shared__.
__device__ __forceinline__ int64_t work_first(unsigned long long *work, long long *slot) {
    if (!work) return blockIdx.x;
    if (threadIdx.x == 0) *slot = (long long)atomicAdd(work, 1ull);
    __syncthreads();
    return *slot;
}
__device__ __forceinline__ int64_t work_next(unsigned long long *work, long long *slot,
                                             int64_t cur) {
    if (!work) return cur + gridDim.x;
    __syncthreads();  // every thread has read the current item
    if (threadIdx.x == 0) *slot = (long long)atomicAdd(work, 1ull);
    __syncthreads();
    return *slot;
}

struct SegArgs {
    int32_t wb;            // window bits per warp bitmap (1024 * S)
    int32_t nwin;          // windows per row
    int32_t seg;           // bitmap words per lane segment (wb / 1024, odd)
    int32_t warp_words;    // shared words per warp (see k_fill_seg)
    int32_t desc_cap;      // descriptor slots (mask words per window)
    int32_t warps;         // warps per block
    const int32_t *bnd;    // (P, nwin+1) members of each bucket below each window start
};

struct BlkArgs {
    int32_t threads;       // threads per CTA (one row per CTA)
    int32_t groups;        // 128-id groups per thread (power of two <= 16)
    int32_t wb;            // window ids = threads * groups * 128
    int32_t nwin;          // windows per row
    int32_t dcap;          // descriptor slots in shared memory (multiple of 8)
    int32_t lcap;          // color slots (>= longest list)
    int32_t nga;           // bitmap groups held in shared memory (multiple of groups)
    int32_t ecap;          // admitted-id list capacity per window (0: always re-decode)
    const int32_t *bnd;    // (P, nwin+1) members of each bucket below each window start
};

struct BinArgs {
    int32_t threads;       // threads per CTA (one row per CTA)
    int32_t shift;         // bins of 2^shift ids
    int32_t nbins;
    int32_t ecap;          // admitted ids per row held in shared memory (>= longest row)
    int32_t dcap;          // descriptor slots (multiple of 8)
    int32_t lcap;          // color slots (>= longest list)
};

struct BucketArgs {
    int64_t P;
    const int32_t *bstart;    // (P+1) bucket bounds in the sorted entry array
    const int32_t *sorted_e;  // list-entry index of every sorted position
    const int32_t *row_of;    // row of every list entry
    const int32_t *bpos;      // (P+1) padded bucket starts
    const int64_t *maskoff;   // (P+1)
    int32_t *bmemp;           // out: padded members
    int32_t *bmem;            // out: unpadded members (direct mode), may be null
    int32_t *posof;           // out: position of each entry in its bucket
    uint32_t *masks;          // out: commute masks
    const uint32_t *A;
    const uint32_t *B;
    int32_t kw;
};

// Launchers (each returns the number of kernels it launched).
int launch_encode(const uint64_t *words, int32_t nwords, const int64_t *active, int64_t n,
                  int64_t npad, int32_t q, int raw, uint32_t *A, uint32_t *B, int32_t kw,
                  int32_t *bad, cudaStream_t s);
int launch_lists(const int64_t *lists, const int64_t *loff, int64_t n, int32_t L,
                 int64_t entries, int64_t base, int64_t P, int32_t *lrel, int32_t *row_of,
                 int32_t *bad, cudaStream_t s);
int launch_bucket_bounds(const int32_t *sorted_colors, const int32_t *eidx, const int32_t *row_of,
                         int64_t entries, int64_t P, int32_t *bstart, int32_t *bad, cudaStream_t s);
int launch_commute_direct(const uint32_t *A, const uint32_t *B, int32_t kw, int64_t npad,
                          int64_t tile0, int64_t tile1, unsigned long long *anti, int sms,
                          cudaStream_t s);
bool fr8_supported(int32_t kw);
// visit order of the 8-bit K1's partner blocks: 0, njb-1, 1, njb-2, ... (a permutation)
__host__ __device__ inline int64_t fr8_fold(int64_t v, int64_t njb) {
    return (v & 1) ? njb - 1 - (v >> 1) : (v >> 1);
}
int fr8_jb(int32_t kw);
int launch_commute_fr8_items(const uint32_t *A, const uint32_t *B, int32_t kw, int64_t n,
                             const int64_t *item_start, int64_t njb, int32_t ichunk,
                             int64_t item0, int64_t item1, unsigned long long *anti, int sms,
                             int warps, cudaStream_t s);
int launch_rows(const RowArgs &a, bool fill, bool out64, int sms, cudaStream_t s);
int launch_bucket_layout(const BucketArgs &b, int64_t entries, cudaStream_t s);
int launch_bucket_masks(const BucketArgs &b, int sms, cudaStream_t s);
size_t owned_masks_smem(const OwnArgs &o, int kw);
int64_t owned_bitmap_words(const OwnArgs &o);
int64_t owned_hash_coll();
int launch_owned_masks(const BucketArgs &b, const OwnArgs &o, int sms, cudaStream_t s);
int launch_count_owned(const RowArgs &a, int sms, cudaStream_t s);
int launch_assign_lists(const int64_t *active, int64_t n, uint64_t base_key, int64_t P, int L,
                        int64_t palette_base, int64_t *out, cudaStream_t s);
void seg_geometry(int64_t n, int64_t max_bits, int32_t *wb, int32_t *nwin, int32_t *seg);
int launch_window_bounds(const int32_t *bstart, const int32_t *bpos, const int32_t *bmemp,
                         int64_t P, int nwin, int32_t wb, int32_t *bnd, cudaStream_t s);
size_t bins_smem_bytes(const BinArgs &g);
void bins_geometry(int64_t n, double mean_deg, int threads, BinArgs *g);
int launch_fill_bins(const RowArgs &a, const BinArgs &g, bool out64, int sms, cudaStream_t s);
size_t blk_smem_bytes(const BlkArgs &g, int groups);
void blk_geometry(int64_t n, int threads, int groups, BlkArgs *g);
int launch_fill_blk(const RowArgs &a, const BlkArgs &g, bool out64, int sms, cudaStream_t s);
int launch_fill_seg(const RowArgs &a, const SegArgs &g, bool out64, int sms, cudaStream_t s);
int launch_widen(const int32_t *src, int64_t *dst, int64_t count, int sms, cudaStream_t s);
int launch_delta(bool write, bool wide, const int32_t *nbr, const int64_t *rowoff, int64_t rows,
                 void *bytes, int32_t *xcount, const int64_t *xoff, int32_t *xval, int sms,
                 cudaStream_t s);
int launch_class_keys(const int64_t *color, int64_t n, int64_t *keys, int32_t *vals, cudaStream_t s);
int launch_class_pairs(bool emit, const int64_t *keys, const int32_t *vals, int64_t n,
                       const uint32_t *A, const uint32_t *B, int32_t kw, int64_t *cnt,
                       const int64_t *off, int64_t cap, int64_t *pairs, cudaStream_t s);
int launch_compact(const int32_t *deg, int64_t n, const int32_t *compact, const int64_t *rowoff,
                   const int64_t *active, int64_t *members_out, int64_t *offsets_out,
                   int32_t *mrow, cudaStream_t s);

// Tile arithmetic shared by host and kernels.
__host__ __device__ inline int64_t tri_tiles(int64_t T) { return T * (T + 1) / 2; }

}  // namespace pcg

struct pcg_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    std::string err;

    // staged inputs
    int64_t n_total = 0, n = 0, npad = 0;
    int32_t nwords = 0, q = 0, L = 0, kw = 0, lmax = 0;
    int64_t base = 0, P = 0, entries = 0;
    bool ragged = false, raw = false, staged = false;

    // options
    int k1_algo = 0;    // 0 auto, 1 direct, 2 four-Russians
    int64_t own_lo = 0, own_hi = -1;  // options own_rows_lo/hi: rows whose owned-mask rows
                                      // the prep computes (-1: all; sharded builds)
    int64_t prep_lo = 0, prep_hi = 0; // the range the current masks hold
    int window = 0;     // K2 window bits (0 auto)
    int fr_ichunk = 0;  // four-Russians i-chunk (0 auto)
    int fill_algo = 0;  // owned masks: 0 auto (block fill up to 128K ids, else the bins fill
                        // when the longest row fits its list (16K ids), else segmented), 7 bins fill
                        // (counting sort per row), 5 block fill (CTA per row), 6 segmented fill (warp-decoded words,
                        // lane-segment harvest), 3 lane-per-bucket bitmap fill (also the fill of
                        // lists longer than 64 colors and of the non-owned mask modes)
    int seg_bits = 0;   // segmented fill: max window bits per warp (0 auto)
    int seg_warps = 0;  // segmented fill: warps per block (0 auto)
    int own_algo = 0;   // owned masks: 0 four-Russians tables (when kw allows), 1 per-pair
    int own_bitmap = 1;   // ownership: exact color bitmap when smaller than the hash table
    int own_direct = 1; // ownership: 1 direct-mapped color table when P is small, 0 hash
    int k2_mode = 0;    // 0 auto, 1 partner gathers, 2 bucket masks + bitmap dedupe, 3 owned masks

    // state of the last count
    bool counted = false;
    int64_t cnt_row_begin = 0, cnt_row_end = 0;
    pcg_counts last{};

    // profiling
    bool prof = false;
    cudaEvent_t ev[12] = {};
    float ktimes[5] = {0, 0, 0, 0, 0};
    void *stage[2] = {nullptr, nullptr};  // pinned D2H staging (32 MiB each)

    // device buffers
    pcg::DevBuf words, active, lists64, loff, A, B, lrel, rowof, keys2, vals2, bstart,
        cubtmp, deg, degu, compact, rowoff, scal, bad, members_o, offsets_o, nbr_o, gdeg, items,
        eidx, bpos, bmemp, posof, maskoff, masks;
    int prep_launches = 0;
    bool masked = false;  // K2 uses bucket masks (K2a/K2b) instead of partner gathers
    bool owned = false;   // masks keep each pair only in its smallest shared color
    int32_t maxdeg = 0;
    int32_t m_max = 0;        // largest color bucket of the staged build
    size_t free_mem = 0;      // device free memory, queried once per context
    bool own_check = false;   // ownership overflow flag still to be read (count pass)
    bool prep_timed = false;  // prep events recorded, elapsed time pending
    int64_t mask_words = 0;   // owned/bucket mask words of the staged build
    pcg::DevBuf bnd;          // segmented fill window bounds
    pcg::DevBuf vcolor, vkeys, vkeys2, vvals, vvals2, vcnt, voff, vpairs;  // validator
    // multi-GPU exchange through peer memory: this rank's exported buffer (the root's CSR
    // ids, written by every rank's fill) and the peers' buffers mapped here
    pcg::DevBuf xbuf;
    pcg::DevBuf workctr;  // atomic work counters of the dynamically scheduled kernels
    int dyn_work = 1;     // K2a and the bins fill take their items from an atomic counter
    int fuse_deg = 1;     // the owned-mask kernel computes the degrees (no K2c pass)
    bool deg_fused = false;  // this prep's degrees came from the owned-mask kernel
    int k1_warps = 0;     // K1 CTA size: 0 auto (8 warps next to the row passes, else 16)
    int k1_shard = 0, k1_nshards = 1;  // the K1 shard an early launch sweeps (sharded build)
    int64_t k1_early_pairs = 0;        // pairs of that shard
    cudaIpcMemHandle_t xhandle{};
    void *xhandle_of = nullptr;  // the allocation xhandle was taken from
    std::vector<std::pair<std::string, void *>> xmaps;  // handle bytes -> mapped pointer
    // pipelined D2H of the neighbor ids: ring of pinned staging chunks
    int d2h_chunk = 0;        // ids per chunk (0 auto)
    int d2h_threads = 0;      // host widening threads (0 auto)
    int d2h_mode = 0;         // 0 byte-delta copy-out; 3 direct int32 copy into pinned
                              // memory; 4 staged int32 copy; 1/2 diagnostics (copies /
                              // widening only, staged path)
    std::vector<void *> ring;
    size_t ring_bytes = 0;
    std::vector<cudaEvent_t> ring_ev;
    std::vector<cudaStream_t> ring_st;
    std::vector<cudaEvent_t> chunk_ev;  // direct D2H: one event per chunk
    int64_t copy_bytes = 0;                    // D2H bytes of the last pcg_fill
    int d2h_gap16 = 0;  // delta copy-out gap width: 0 auto (mean gap), 1 16-bit, 2 bytes
    int d2h_pipe = 1;   // public build: fill in pieces overlapping the copy-out (0 = off)
    int d2h_pieces = 0; // pieces of the pipelined fill (0 auto)
    int d2h_dma = -1;   // % of copy-out chunks sent as int64 by DMA into a pinned output (-1 auto)
    pcg::DevBuf dwide;  // device int64 staging of those chunks
    cudaStream_t dma_st = nullptr;
    pcg::DevBuf mrow;   // member -> active row (pipelined fill)
    std::vector<cudaEvent_t> piece_ev;
    cudaEvent_t scan_ev = nullptr;
    std::vector<std::pair<int32_t *, size_t>> hxpiece;  // pinned exceptions per piece
    int blk_threads = 0, blk_groups = 0, blk_dcap = 0, blk_ecap = 0;  // block fill geometry (0 = auto)
    unsigned char *hs = nullptr;  // pinned scratch for the small per-build readbacks (512 B)
    int64_t launch_total = 0;     // kernels launched by this context (pcg_launch_total)
    int rows_out32 = 0;           // pcg_fill_rows_device writes int32 ids (sharded exchange)
    int rows_out_abs = 0;         // ... at the rows' global CSR offsets (peer exchange buffer)
    int k1_early = 2;  // K1 from the input prep (1), from the count pass (0), auto (2)
    bool k1_early_valid = false;  // an early K1 of the staged build is in flight (scal[7])
    int k1_slot = 0;              // scal word pcg_k1_result reads (0, or 7 for the early K1)
    int bins_threads = 0;  // bins fill: threads per CTA (0 = auto)
    int bins_shift = 0;    // bins fill: bin width exponent delta from auto (testing/tuning)
    int bins_maxdeg = 0;   // bins fill: longest row it takes (0 = 16384)
    int k1_async = 0;                          // K1 on a side stream, result collected later
    bool k1_pending = false;
    cudaStream_t k1_stream = nullptr;
    cudaEvent_t k1_fork = nullptr, k1_done = nullptr;
    pcg::DevBuf dbytes, dxcnt, dxoff, dxval;  // byte-delta encoded CSR (public-build copy-out)
    std::vector<uint8_t *> hbytes;             // pinned per-worker byte staging
    size_t hbytes_cap = 0;
    int32_t *hxval = nullptr;                  // pinned exceptions + per-row offsets
    int64_t *hxoff = nullptr;
    size_t hx_cap = 0, hxoff_cap = 0;
};
