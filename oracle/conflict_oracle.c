/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference conflict-graph builder
 * (palettecolor.conflict.build, /root/reference/pkg/src/palettecolor/conflict.py:89-167).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg may load this library, and only as the checker or as the timed CPU baseline.
 * The product path (paper_2401_06713_b200) never links, imports or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks every function here against the golden
 * vectors in tests/golden/ (produced by tools/make_golden.py from the reference
 * itself, imported in the build container).
 *
 * What each routine follows:
 *   anticommute()        pauli.py:258-268 (anticommute_pairs: XOR-accumulated popcount
 *                        parity of words[i] & words[j]); graph.py:335-336 (implicit
 *                        complement edge = NOT anticommute).
 *   make_masks()         driver.py:152-172 (ColorLists.mask_matrix: dense palette bitmask
 *                        relative to palette_base, ceil(P/64) uint64 words per vertex).
 *   intersect()          conflict.py:77 ((masks[i] & masks[j]).any(axis=1)).
 *   oracle_build_count   conflict.py:110-118 (two-phase count: admitted and oracle-edge
 *                        counts over the upper triangle; block order == row-major order,
 *                        graph.py:379-407).
 *   oracle_build_fill    conflict.py:119-130 (fill u/v arrays in block order).
 *   oracle_csr_assemble  conflict.py:148-161 (union1d / searchsorted / lexsort / add.at /
 *                        cumsum).  Appending each admitted (u,v) to both rows while walking
 *                        the pairs in row-major order yields exactly the lexsort order: row r
 *                        receives its w<r entries first (ascending w) then its v>r entries
 *                        (ascending v).
 *   oracle_row           one full conflict row (both directions) — the same predicate as
 *                        above, used for sampled-row checks where the full build is too big.
 *   oracle_commute_count conflict.py:78,115 (view_edges_scanned = #commuting pairs).
 *
 * Threads only split rows; all outputs are independent of the thread count
 * (conflict.py:81-86 merges blocks in block order; we write per-row prefix offsets).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const uint64_t *words;   /* (n_total, nwords) packed 3-bit Pauli words */
    int64_t nwords;
    const int64_t *active;   /* (n,) sorted original ids */
    int64_t n;
    const uint64_t *masks;   /* (n, mwords) palette bitmasks, or NULL when only commuting */
    int64_t mwords;
    /* outputs */
    int64_t *deg_upper;      /* count pass: admitted j>i per row */
    int64_t *seen_upper;     /* count pass: commuting j>i per row */
    const int64_t *row_pos;  /* fill pass: prefix of deg_upper */
    int64_t *v_arr;          /* fill pass output */
    /* scheduling */
    int64_t next_row;
    pthread_mutex_t lock;
    int mode;                /* 0 count, 1 fill, 2 commute-count only */
} job_t;

static inline int anticommute(const uint64_t *a, const uint64_t *b, int64_t nw) {
    uint64_t acc = 0;
    for (int64_t w = 0; w < nw; ++w) acc ^= a[w] & b[w];
    return __builtin_parityll(acc);
}

static inline int intersect(const uint64_t *a, const uint64_t *b, int64_t mw) {
    for (int64_t w = 0; w < mw; ++w)
        if (a[w] & b[w]) return 1;
    return 0;
}

static int64_t grab_rows(job_t *jb, int64_t chunk, int64_t *lo) {
    pthread_mutex_lock(&jb->lock);
    *lo = jb->next_row;
    int64_t hi = *lo + chunk;
    if (hi > jb->n) hi = jb->n;
    jb->next_row = hi;
    pthread_mutex_unlock(&jb->lock);
    return hi;
}

static void *worker(void *arg) {
    job_t *jb = (job_t *)arg;
    const int64_t nw = jb->nwords, mw = jb->mwords;
    for (;;) {
        int64_t lo, hi = grab_rows(jb, 16, &lo);
        if (lo >= hi) break;
        for (int64_t i = lo; i < hi; ++i) {
            const uint64_t *wi = jb->words + jb->active[i] * nw;
            const uint64_t *mi = jb->masks ? jb->masks + i * mw : NULL;
            int64_t adm = 0, seen = 0;
            int64_t pos = (jb->mode == 1) ? jb->row_pos[i] : 0;
            for (int64_t j = i + 1; j < jb->n; ++j) {
                const uint64_t *wj = jb->words + jb->active[j] * nw;
                if (anticommute(wi, wj, nw)) continue;
                ++seen;
                if (jb->mode == 2) continue;
                if (!intersect(mi, jb->masks + j * mw, mw)) continue;
                if (jb->mode == 1) jb->v_arr[pos + adm] = j;
                ++adm;
            }
            if (jb->mode != 1) {
                if (jb->deg_upper) jb->deg_upper[i] = adm;
                jb->seen_upper[i] = seen;
            }
        }
    }
    return NULL;
}

static void run_job(job_t *jb, int threads) {
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    jb->next_row = 0;
    pthread_mutex_init(&jb->lock, NULL);
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, worker, jb);
    worker(jb);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&jb->lock);
}

/* driver.py:152-172: rows given as CSR (list_off) so ragged ColorLists work too.
 * Returns 0, or -1 on a color outside [base, base+P). */
int oracle_make_masks(const int64_t *list_data, const int64_t *list_off, int64_t n,
                      int64_t palette_base, int64_t palette_size, uint64_t *masks) {
    int64_t mw = palette_size > 0 ? (palette_size + 63) / 64 : 1;
    memset(masks, 0, (size_t)(n * mw) * sizeof(uint64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t k = list_off[i]; k < list_off[i + 1]; ++k) {
            int64_t rel = list_data[k] - palette_base;
            if (rel < 0 || rel >= mw * 64) return -1;
            masks[i * mw + (rel >> 6)] |= 1ULL << (rel & 63);
        }
    return 0;
}

int64_t oracle_mask_words(int64_t palette_size) {
    return palette_size > 0 ? (palette_size + 63) / 64 : 1;
}

/* conflict.py:110-118 */
int oracle_build_count(const uint64_t *words, int64_t nwords, const int64_t *active,
                       int64_t n, const uint64_t *masks, int64_t mwords, int threads,
                       int64_t *deg_upper, int64_t *seen_upper) {
    job_t jb;
    memset(&jb, 0, sizeof jb);
    jb.words = words; jb.nwords = nwords; jb.active = active; jb.n = n;
    jb.masks = masks; jb.mwords = mwords;
    jb.deg_upper = deg_upper; jb.seen_upper = seen_upper; jb.mode = 0;
    run_job(&jb, threads);
    return 0;
}

/* conflict.py:119-130 */
int oracle_build_fill(const uint64_t *words, int64_t nwords, const int64_t *active,
                      int64_t n, const uint64_t *masks, int64_t mwords, int threads,
                      const int64_t *row_pos, int64_t *v_arr) {
    job_t jb;
    memset(&jb, 0, sizeof jb);
    jb.words = words; jb.nwords = nwords; jb.active = active; jb.n = n;
    jb.masks = masks; jb.mwords = mwords;
    jb.row_pos = row_pos; jb.v_arr = v_arr; jb.mode = 1;
    run_job(&jb, threads);
    return 0;
}

/* conflict.py:78,115 without the list test: the number of commuting pairs. */
int64_t oracle_commute_count(const uint64_t *words, int64_t nwords, const int64_t *active,
                             int64_t n, int threads) {
    job_t jb;
    memset(&jb, 0, sizeof jb);
    int64_t *seen = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    jb.words = words; jb.nwords = nwords; jb.active = active; jb.n = n;
    jb.seen_upper = seen; jb.mode = 2;
    run_job(&jb, threads);
    int64_t total = 0;
    for (int64_t i = 0; i < n; ++i) total += seen[i];
    free(seen);
    return total;
}

/* conflict.py:148-161.  row_pos: (n+1) prefix of deg_upper; v_arr: upper-triangle partner
 * of each admitted pair in row-major order (u is implied by row_pos).
 * Outputs: members (local ids, caller maps through active), offsets (n_members+1),
 * neighbors (2*E).  Returns n_members. */
int64_t oracle_csr_assemble(int64_t n, const int64_t *row_pos, const int64_t *v_arr,
                            int64_t *members_local, int64_t *offsets, int64_t *neighbors) {
    int64_t E = row_pos[n];
    int64_t *deg = (int64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(int64_t));
    int64_t *cid = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    for (int64_t u = 0; u < n; ++u)
        for (int64_t e = row_pos[u]; e < row_pos[u + 1]; ++e) {
            ++deg[u];
            ++deg[v_arr[e]];
        }
    int64_t nm = 0;
    for (int64_t u = 0; u < n; ++u) {
        cid[u] = deg[u] ? nm : -1;
        if (deg[u]) members_local[nm++] = u;
    }
    offsets[0] = 0;
    for (int64_t k = 0; k < nm; ++k) offsets[k + 1] = offsets[k] + deg[members_local[k]];
    int64_t *fillp = (int64_t *)malloc((size_t)(nm > 0 ? nm : 1) * sizeof(int64_t));
    for (int64_t k = 0; k < nm; ++k) fillp[k] = offsets[k];
    for (int64_t u = 0; u < n; ++u)
        for (int64_t e = row_pos[u]; e < row_pos[u + 1]; ++e) {
            int64_t cu = cid[u], cv = cid[v_arr[e]];
            neighbors[fillp[cu]++] = cv;
            neighbors[fillp[cv]++] = cu;
        }
    (void)E;
    free(fillp);
    free(cid);
    free(deg);
    return nm;
}

/* One full conflict row of local vertex i (ascending local ids j != i), plus the number of
 * vertices commuting with i.  out must hold n entries.  Returns the row length. */
int64_t oracle_row(const uint64_t *words, int64_t nwords, const int64_t *active, int64_t n,
                   const uint64_t *masks, int64_t mwords, int64_t i, int64_t *out,
                   int64_t *commuting) {
    const uint64_t *wi = words + active[i] * nwords;
    const uint64_t *mi = masks + i * mwords;
    int64_t len = 0, seen = 0;
    for (int64_t j = 0; j < n; ++j) {
        if (j == i) continue;
        if (anticommute(wi, words + active[j] * nwords, nwords)) continue;
        ++seen;
        if (intersect(mi, masks + j * mwords, mwords)) out[len++] = j;
    }
    *commuting = seen;
    return len;
}

/* Time-boxed CPU baseline: the reference's per-pair work (predicate + dense palette AND,
 * conflict.py:72-78) over rows [row_lo, row_hi) of the upper triangle.  Returns admitted
 * pairs; *pairs_out = pairs scanned. */
int64_t oracle_scan_rows(const uint64_t *words, int64_t nwords, const int64_t *active,
                         int64_t n, const uint64_t *masks, int64_t mwords, int64_t row_lo,
                         int64_t row_hi, int64_t *pairs_out, int64_t *seen_out) {
    int64_t adm = 0, seen = 0, pairs = 0;
    for (int64_t i = row_lo; i < row_hi && i < n; ++i) {
        const uint64_t *wi = words + active[i] * nwords;
        const uint64_t *mi = masks + i * mwords;
        for (int64_t j = i + 1; j < n; ++j) {
            ++pairs;
            int edge = !anticommute(wi, words + active[j] * nwords, nwords);
            /* conflict.py:77 evaluates the mask AND for every pair of the block; this port
             * stops at the first shared word, which only makes the baseline faster */
            int inter = intersect(mi, masks + j * mwords, mwords);
            seen += edge;
            adm += edge & inter;
        }
    }
    *pairs_out = pairs;
    *seen_out = seen;
    return adm;
}
