/*
 * picasso_b200.h — C ABI of the B200 conflict-graph builder.
 *
 * Drop-in target: palettecolor.conflict.build(view, lists, *, edge_budget, threads,
 * block_pairs, two_phase) -> ConflictGraph
 *   (/root/reference/pkg/src/palettecolor/conflict.py:89-167).
 * The reference has no FFI of its own (pure Python + numpy); these entry points are what a
 * ctypes / cffi binding of that function binds — see INTEGRATION.md.  Plain pointers and
 * sizes only; no torch types; no exceptions cross the ABI (every call returns a status).
 *
 * The two-phase contract of the reference (count -> budget check -> fill) is kept:
 *   pcg_set_inputs   conflict.py:106-108   inputs of one build (words, active ids, lists)
 *   pcg_count        conflict.py:110-116   count pass: degrees, |E_c|, view_edges_scanned
 *                                          (the budget check, conflict.py:117-118, is the
 *                                          caller's: it raises EdgeBudgetExceededError)
 *   pcg_fill         conflict.py:119-161   fill pass + canonical CSR (members, offsets,
 *                                          neighbors) written straight into caller buffers
 * and, for pair-space sharding across GPUs (one process per GPU, host collectives):
 *   pcg_copy_degrees / pcg_fill_rows       per-shard degrees out, global degrees in, shard
 *                                          slice of the CSR out.
 *
 * Thread safety: one pcg_ctx per host thread; contexts share nothing.
 */
#ifndef PICASSO_B200_H
#define PICASSO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PCG_OK 0
#define PCG_E_ARG 1      /* bad argument (null pointer, size out of range, bad qubit count) */
#define PCG_E_CUDA 2     /* CUDA runtime error (see pcg_last_error) */
#define PCG_E_OOM 3      /* device allocation failed */
#define PCG_E_COLOR 4    /* a list color lies outside [palette_base, palette_base + palette_size) */
#define PCG_E_STATE 5    /* call order violated (fill before count, ...) */
#define PCG_E_DUPLICATE 6 /* a row's color list names one color twice (the caller dedupes: the
                             reference's palette mask is a set, driver.py:152-172) */

typedef struct pcg_ctx pcg_ctx;

/* Totals of one count pass (conflict.py:114-116). */
typedef struct {
    int64_t n_active;           /* rows of the build (view.n_active) */
    int64_t anticommuting;      /* anticommuting pairs among the K1 tile shard */
    int64_t pairs_in_shard;     /* unordered pairs covered by the K1 tile shard */
    int64_t deg_sum;            /* sum of conflict degrees over the K2 row range */
    int64_t deg_upper_sum;      /* sum over the row range of #admitted partners j > i */
    int64_t members_in_range;   /* rows of the range with degree > 0 */
    int32_t raw_words_mode;     /* 1 if invalid 3-bit codes forced the raw-word predicate */
    int32_t reserved;
} pcg_counts;

int pcg_version(void);
/* Creates a context bound to CUDA device `device` with its own stream. */
int pcg_create(int device, pcg_ctx **out);
int pcg_destroy(pcg_ctx *ctx);
const char *pcg_last_error(const pcg_ctx *ctx);

/*
 * Stage the inputs of one build (host pointers, copied to the device).
 *   words      (n_total, nwords) uint64: PauliSet.words (pauli.py:217, 240-246)
 *   active     (n_active,) int64, sorted unique original ids (graph.py:291-303)
 *   list_data  colors of every active row, row-major (ColorLists.array, driver.py:184-188)
 *   list_off   (n_active+1,) int64 row offsets into list_data, or NULL when every row has
 *              exactly list_len colors (the rectangular ColorLists.array case)
 *   palette_base / palette_size: ColorLists.palette_base / palette_size
 */
int pcg_set_inputs(pcg_ctx *ctx, const uint64_t *words, int64_t n_total, int32_t nwords,
                   int32_t num_qubits, const int64_t *active, int64_t n_active,
                   const int64_t *list_data, const int64_t *list_off, int32_t list_len,
                   int64_t palette_base, int64_t palette_size);

/*
 * Count pass.  The commuting-pair count (view_edges_scanned) runs over tile shard
 * `shard` of `nshards` of the upper triangle; conflict degrees are computed for full
 * rows [row_begin, row_end).  Single GPU: shard=0, nshards=1, rows [0, n_active).
 * view_edges_scanned = pairs - anticommuting (summed over shards); |E_c| = deg_sum / 2
 * (summed over row ranges).
 */
int pcg_count(pcg_ctx *ctx, int32_t shard, int32_t nshards, int64_t row_begin,
              int64_t row_end, pcg_counts *out);

/* Degrees of rows [row_begin,row_end) from the last count: deg (full row) and deg_upper
 * (partners j > i), int32 host buffers of (row_end-row_begin) entries; either may be NULL. */
int pcg_copy_degrees(pcg_ctx *ctx, int32_t *deg, int32_t *deg_upper);

/*
 * Fill pass + CSR for the single-GPU case (count must cover all rows).  Host outputs,
 * int64 like the reference: members (n_members), offsets (n_members+1),
 * neighbors (2*edge_count).  n_members = rows with degree > 0.
 */
int pcg_fill(pcg_ctx *ctx, int64_t *members, int64_t *offsets, int64_t *neighbors);

/*
 * Sharded fill.  global_deg: (n_active,) int32 degrees of ALL rows (gathered from every
 * shard, host pointer).  Writes the neighbor entries of rows [row_begin,row_end) — a
 * contiguous slice of the global CSR neighbor array starting at entry *slice_begin —
 * into `neighbors` (host, int64, capacity (*slice_end - *slice_begin)).
 * Call with neighbors == NULL first to learn the slice bounds.
 */
int pcg_fill_rows(pcg_ctx *ctx, const int32_t *global_deg, int64_t *neighbors,
                  int64_t *slice_begin, int64_t *slice_end);

/* Sharded build with device pointers (the NCCL merge operates on the caller's device
 * buffers): degrees of the counted row range into deg_dev (int32, row_end-row_begin); the
 * rows' CSR slice into neighbors_dev (int64; call with NULL first to learn the bounds). */
int pcg_degrees_device(pcg_ctx *ctx, int32_t *deg_dev);
/* Re-run the device input prep (bit planes, color buckets, bucket masks) on the staged raw
 * inputs — the per-step replicated work of a sharded build. */
int pcg_prep_device(pcg_ctx *ctx);
int pcg_fill_rows_device(pcg_ctx *ctx, const int32_t *global_deg_dev, int32_t maxdeg,
                         int64_t *neighbors_dev, int64_t *slice_begin, int64_t *slice_end);
/* (With pcg_set_option(ctx, "rows_out32", 1) neighbors_dev receives int32 ids instead: the
 * sharded build exchanges half the bytes and widens after the all-gather.) */

/* Device-resident timing hooks for the benchmark (no host traffic): re-run count and fill
 * on the inputs already staged; outputs stay in HBM.  *launches receives the number of
 * kernels this call launched. */
int pcg_count_device(pcg_ctx *ctx, pcg_counts *out, int32_t *launches);
int pcg_fill_device(pcg_ctx *ctx, int32_t *launches);
/* One whole build on the staged raw inputs, device only: input prep (bit planes, color
 * buckets, bucket commute masks) + count + fill; the CSR stays in HBM. */
int pcg_build_device(pcg_ctx *ctx, pcg_counts *out, int32_t *launches);
/* Average device time (ms) of each kernel family in the last *_device call:
 * [0] commute sweep (K1), [1] conflict-row count (K2c), [2] conflict-row fill (K2f),
 * [3] compaction/offsets, [4] input prep.  Requires pcg_set_profiling(ctx, 1). */
int pcg_set_profiling(pcg_ctx *ctx, int32_t on);
/* The context's CUDA stream (cudaStream_t), so callers can time it with their own events. */
void *pcg_stream(pcg_ctx *ctx);
int pcg_kernel_times(pcg_ctx *ctx, float *ms, int32_t n);
/* Kernel configuration knobs (testing/tuning; 0 = auto unless noted).  Every setting gives
 * the same CSR; the defaults are the measured fastest.
 *   K1 (commuting pairs):  "k1_algo" 1 direct LOP3/POPC tiles, 5 four-Russians 8-bit slices
 *                          (default for q <= 128); "fr_ichunk" rows per work item; "k1_async"
 *                          1 runs K1 on a side stream (pcg_k1_result collects it); "k1_early"
 *                          with k1_async: 1 from the input prep (beside the owned masks), 0
 *                          from the count pass, 2 (default) prep from 256K rows; "k1_warps"
 *                          CTA size (0: 8 warps beside other kernels, else 16); "dyn_work" 1
 *                          (default) owned masks and bins fill take items from atomic counters
 *   K2 (conflict rows):    "k2_mode" 1 partner gather, 2 bucket masks, 3 owned masks;
 *                          "own_algo" 0 four-Russians / 1 per-pair masks; "own_direct" 0 turns
 *                          off the direct-mapped ownership table (small palettes); "own_bitmap"
 *                          0 turns off the exact color bitmap (then the hash table);
 *                          "window" row-pass bitmap (ids)
 *   fill:                  "fill_algo" 0 auto, 3 lane bitmap, 5 block (CTA per row),
 *                          6 segmented, 7 bins (counting sort);
 *                          "blk_threads" "blk_groups" "blk_dcap" "blk_ecap"; "bins_threads"
 *                          "bins_shift" "bins_maxdeg"; "seg_bits" "seg_warps"
 *   copy-out (pcg_fill):   "d2h_mode" 0 delta gaps (default) / 3 direct / 4 int32 widen;
 *                          "d2h_pipe" 1 (default) fill in pieces overlapping the copy-out,
 *                          "d2h_pieces", "d2h_chunk" (ids), "d2h_threads", "d2h_gap16"
 *                          (1 16-bit, 2 8-bit gaps), "d2h_dma" (% of chunks as int64 DMA)
 *   sharded:               "rows_out32" 1: pcg_fill_rows_device writes int32 ids;
 *                          "rows_out_abs" 1: ... at the rows' global CSR offsets (the
 *                          pointer is the whole CSR's base: the root's exchange buffer) */
int pcg_set_option(pcg_ctx *ctx, const char *key, int64_t value);

/*
 * Palette lists on the device (rng.py:22-70 + driver.py:175-188, bit-identical): for each
 * active id v, list_size distinct colors of [0, palette_size) by Floyd sampling on the
 * splitmix64 stream mix64(v*phi + base_key), sorted, + palette_base.  base_key =
 * mix64(seed + phi*iteration) (rng.stream_keys).  out: (n, list_size) int64, host.
 */
int pcg_assign_lists(pcg_ctx *ctx, const int64_t *active, int64_t n, uint64_t base_key,
                     int64_t palette_size, int32_t list_size, int64_t palette_base, int64_t *out);

/*
 * Host list coloring of a conflict CSR, dynamic bucket scheme (list_coloring.py:53-139),
 * draw-for-draw identical to numpy's Generator(PCG64).  rng6 = {state_hi, state_lo, inc_hi,
 * inc_lo, has_uint32, uinteger} (numpy's PCG64 state), advanced in place.  color_of[k] =
 * chosen color of member k, or INT64_MIN for the uncolored residue.
 */
int pcg_color_dynamic(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                      const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                      int64_t *color_of, int64_t *removal_ops);
/* Same coloring (same draws, same result).  par_min_deg >= -1 (default -1): each step walks
 * the picked color's bucket (members listing it, ascending) and tests adjacency by galloping
 * through the CSR row; par_min_deg < -1: the neighbor-row scan split across `threads` host
 * threads (0: up to 16) for rows of at least -par_min_deg-2 entries, hits applied in row order
 * (also taken when the colors do not suit buckets).  pcg_color_dynamic = (0, -1). */
int pcg_color_dynamic_mt(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                         const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                         int64_t *color_of, int64_t *removal_ops, int32_t threads,
                         int64_t par_min_deg);
/* Same coloring for the conflict graph of a Pauli view, without the CSR: words = the members'
 * packed 3-bit code words (nm x nwords, PauliSet.words[members], pauli.py:217); two members of
 * one color bucket are conflict neighbors iff their strings commute (graph.py:327-336).
 * Returns 1, having drawn nothing, when the colors do not suit the bucket form (color range
 * above 2^28, or a list naming a color twice): use pcg_color_dynamic_mt then.  Both return -2
 * when host memory runs out (no exception crosses the ABI). */
int pcg_color_dynamic_words(int64_t nm, const uint64_t *words, int32_t nwords,
                            const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                            int64_t *color_of, int64_t *removal_ops);

/*
 * Exhaustive properness check of a coloring (validation.py:41-131, exhaustive mode; the
 * reference enumerates all pairs in Python and stops at 20,000 vertices, graph.py:34).
 * words / active as in pcg_set_inputs; color (n_active,) int64: the color of each active
 * vertex, INT64_MIN for uncolored (never a violation).  Outputs: *edges = commuting pairs
 * (|E|, oracle_edges), *violations = commuting pairs with equal colors, and the first
 * min(cap, *violations) of them in the reference's enumeration order (i ascending, then j)
 * as local index pairs into pairs_out (2*cap int64).  Invalidates a staged build.
 */
int pcg_validate(pcg_ctx *ctx, const uint64_t *words, int64_t n_total, int32_t nwords,
                 int32_t num_qubits, const int64_t *active, int64_t n_active,
                 const int64_t *color, int32_t cap, int64_t *pairs_out, int64_t *violations,
                 int64_t *edges);

/*
 * Pin (on=1) or unpin (on=0) a host range with cudaHostRegister.  pcg_fill copies the
 * neighbor ids straight into a pinned destination (no staging buffer); the Python layer
 * registers its reused host output buffer once (hostpool.py).
 */
int pcg_host_register(void *ptr, uint64_t bytes, int32_t on);

/*
 * Multi-GPU exchange through peer memory (replaces the slice gather of a sharded build,
 * SURVEY.md §8(e); the reference has no multi-GPU path — its single build is conflict.py:
 * 89-167).  The root calls pcg_exchange_buffer for a device buffer of `bytes` (reused while
 * large enough) and its 64-byte CUDA IPC handle; every rank maps it with pcg_exchange_map
 * (cached per handle) and passes the mapped pointer to pcg_fill_rows_device with
 * "rows_out32" = 1 and "rows_out_abs" = 1, so its fill stores its rows straight into the
 * root's HBM over NVLink, at their global offsets.  After a barrier the root copies the int32 ids to its int64 host
 * output with pcg_ids_to_host.
 */
int pcg_exchange_buffer(pcg_ctx *ctx, uint64_t bytes, void **dptr, uint8_t *handle);
int pcg_exchange_map(pcg_ctx *ctx, const uint8_t *handle, void **dptr);
int pcg_ids_to_host(pcg_ctx *ctx, const int32_t *src_dev, int64_t count, int64_t *dst);

/*
 * With the option "k1_async" set, pcg_count launches the commuting-pair sweep (K1) on a side
 * stream next to the conflict-row passes and returns anticommuting = -1; this call waits for
 * it and returns the anticommuting count (view_edges_scanned = pairs_in_shard - it).
 * Without the option it returns the count pcg_count already reported.
 */
int pcg_k1_result(pcg_ctx *ctx, int64_t *anticommuting);

/* Bytes the last pcg_fill copied device -> host: members, offsets and the neighbor ids
 * (sent as gaps + an exception list and decoded into the int64 output on the host; 8-bit
 * gaps while the mean gap is <= 64 ids, else 16-bit — option "d2h_gap16": 1 forces 16-bit,
 * 2 forces 8-bit). */
int64_t pcg_last_copy_bytes(const pcg_ctx *ctx);

/* Kernels this context has launched so far (benchmark accounting). */
int64_t pcg_launch_total(const pcg_ctx *ctx);

#ifdef __cplusplus
}
#endif

#endif /* PICASSO_B200_H */
