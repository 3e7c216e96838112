/*
 * ORACLE — TEST INFRASTRUCTURE ONLY (scale oracle).
 *
 * A second plain-C restatement of the reference conflict-graph builder
 * (palettecolor.conflict.build, /root/reference/pkg/src/palettecolor/conflict.py:89-167),
 * written for the sizes where the reference and the dense-mask oracle (conflict_oracle.c)
 * cannot run: configs 2-4 (100k x 32q ... 4M x 128q).  Memory is O(n*L + |E_c|) instead of
 * the reference's O(n * P/64) palette mask plus O(block) index arrays, and the work is
 * O(sum over rows of the row's bucket candidates) instead of O(n^2 * P/64).
 *
 * Same semantics, restated per row:
 *   conflict.py:76-77   pair (i, j) is admitted  <=>  the view has the edge (the pair
 *                       commutes, graph.py:335-336 implicit complement of pauli.py:258-268
 *                       anticommute_pairs) AND (mask_i & mask_j).any().
 *   driver.py:152-172   mask bit r is set  <=>  color palette_base + r is in the row's
 *                       list, 0 <= r < 64*ceil(P/64); duplicated colors OR the same bit.
 *   => (mask_i & mask_j).any()  <=>  the rows share a relative color r in that range.
 *      So row i's conflict partners are exactly the commuting j != i found in the color
 *      buckets of i's colors; a j reached through several shared colors is taken once.
 *   conflict.py:148-161 canonical CSR: members = rows with >= 1 admitted pair, ascending;
 *                       row k lists its partners' compact ids ascending (lexsort order).
 *   conflict.py:78,115  view_edges_scanned = number of commuting pairs (i < j), whatever
 *                       the lists (bk_commute_count).
 *
 * Parity pinning: tests/test_oracle.py checks this oracle against the reference's own golden
 * builds (tests/golden/, made by tools/make_golden.py from the reference itself), the q=32
 * 5k/10k/20k hashes, the c1 per-iteration hashes, and the dense oracle on random ragged /
 * duplicate-color / invalid-code cases.  tools/make_golden_scale.py then uses it to commit
 * the config-2/3/4 iteration-1 CSR hashes and the config-3 whole-run coloring that the GPU
 * tests compare against.
 *
 * Every entry point is thread-safe for distinct output ranges: callers parallelise over row
 * ranges (ctypes releases the GIL).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    const uint64_t *words;   /* (n_total, nwords) packed 3-bit Pauli words (caller-owned) */
    int64_t nwords;
    const int64_t *active;   /* (n,) sorted original ids (caller-owned) */
    int64_t n;
    int64_t ncolors;         /* relative color range: 64 * ceil(P/64) */
    int64_t *bstart;         /* (ncolors + 1) bucket offsets */
    int32_t *bmem;           /* bucket members (local rows, ascending within a bucket) */
    int32_t *rcolors;        /* (n_entries) relative colors of each row, list order */
    int64_t *roff;           /* (n + 1) row offsets into rcolors */
    uint64_t *wloc;          /* (n, nwords) words of the active rows, local order */
    const int64_t *cid;      /* optional local -> compact id map (caller-owned) */
} bk_t;

static inline int anticommute(const uint64_t *a, const uint64_t *b, int64_t nw) {
    uint64_t acc = 0;
    for (int64_t w = 0; w < nw; ++w) acc ^= a[w] & b[w];
    return __builtin_parityll(acc);
}

void bk_close(bk_t *h) {
    if (!h) return;
    free(h->bstart);
    free(h->bmem);
    free(h->rcolors);
    free(h->roff);
    free(h->wloc);
    free(h);
}

/* Buckets: counting sort of (relative color, row) by color; rows ascend inside a bucket
 * because rows are visited in order.  A duplicated color in one row puts the row in the
 * bucket twice; the per-row stamp below takes each partner once (the mask OR semantics).
 * Returns NULL when a color lies outside [base, base + 64*ceil(P/64)) (the reference's
 * mask_matrix would index out of its row) or on allocation failure. */
bk_t *bk_open(const uint64_t *words, int64_t nwords, const int64_t *active, int64_t n,
              const int64_t *list_data, const int64_t *list_off, int64_t palette_base,
              int64_t palette_size) {
    bk_t *h = (bk_t *)calloc(1, sizeof(bk_t));
    if (!h) return NULL;
    h->words = words;
    h->nwords = nwords;
    h->active = active;
    h->n = n;
    h->ncolors = 64 * (palette_size > 0 ? (palette_size + 63) / 64 : 1);
    int64_t ne = list_off[n];
    h->bstart = (int64_t *)calloc((size_t)h->ncolors + 1, sizeof(int64_t));
    h->bmem = (int32_t *)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(int32_t));
    h->rcolors = (int32_t *)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(int32_t));
    h->roff = (int64_t *)malloc((size_t)(n + 1) * sizeof(int64_t));
    h->wloc = (uint64_t *)malloc((size_t)(n > 0 ? n : 1) * (size_t)nwords * sizeof(uint64_t));
    if (!h->bstart || !h->bmem || !h->rcolors || !h->roff || !h->wloc) {
        bk_close(h);
        return NULL;
    }
    for (int64_t i = 0; i <= n; ++i) h->roff[i] = list_off[i];
    for (int64_t e = 0; e < ne; ++e) {
        int64_t rel = list_data[e] - palette_base;
        if (rel < 0 || rel >= h->ncolors) {
            bk_close(h);
            return NULL;
        }
        h->rcolors[e] = (int32_t)rel;
        h->bstart[rel + 1]++;
    }
    for (int64_t c = 0; c < h->ncolors; ++c) h->bstart[c + 1] += h->bstart[c];
    int64_t *pos = (int64_t *)malloc((size_t)h->ncolors * sizeof(int64_t));
    if (!pos) {
        bk_close(h);
        return NULL;
    }
    memcpy(pos, h->bstart, (size_t)h->ncolors * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i)
        for (int64_t e = list_off[i]; e < list_off[i + 1]; ++e)
            h->bmem[pos[h->rcolors[e]]++] = (int32_t)i;
    free(pos);
    for (int64_t i = 0; i < n; ++i)
        memcpy(h->wloc + i * nwords, words + active[i] * nwords, (size_t)nwords * sizeof(uint64_t));
    return h;
}

void bk_set_compact(bk_t *h, const int64_t *cid) { h->cid = cid; }

/* LSD radix sort of uint32 keys (11-bit digits; passes above the top set bit skipped). */
static void radix_sort_u32(uint32_t *a, uint32_t *tmp, int64_t m, uint32_t maxkey) {
    int passes = 1;
    while (passes < 3 && (maxkey >> (11 * passes))) ++passes;
    uint32_t *src = a, *dst = tmp;
    for (int p = 0; p < passes; ++p) {
        int64_t cnt[2049];
        memset(cnt, 0, sizeof cnt);
        int sh = 11 * p;
        for (int64_t k = 0; k < m; ++k) cnt[((src[k] >> sh) & 2047) + 1]++;
        for (int b = 0; b < 2048; ++b) cnt[b + 1] += cnt[b];
        for (int64_t k = 0; k < m; ++k) dst[cnt[(src[k] >> sh) & 2047]++] = src[k];
        uint32_t *t = src;
        src = dst;
        dst = t;
    }
    if (src != a) memcpy(a, src, (size_t)m * sizeof(uint32_t));
}

/* Scratch for one calling thread: a stamp per row (the row that last took it) and the
 * candidate buffers. */
typedef struct {
    int32_t *stamp;
    uint32_t *buf, *tmp;
    int64_t cap;
} scratch_t;

static int scratch_init(scratch_t *s, const bk_t *h) {
    s->stamp = (int32_t *)malloc((size_t)(h->n > 0 ? h->n : 1) * sizeof(int32_t));
    s->cap = 1 << 16;
    s->buf = (uint32_t *)malloc((size_t)s->cap * sizeof(uint32_t));
    s->tmp = (uint32_t *)malloc((size_t)s->cap * sizeof(uint32_t));
    if (!s->stamp || !s->buf || !s->tmp) return -1;
    for (int64_t k = 0; k < h->n; ++k) s->stamp[k] = -1;
    return 0;
}

static void scratch_free(scratch_t *s) {
    free(s->stamp);
    free(s->buf);
    free(s->tmp);
}

/* Conflict partners of local row i (ascending local ids) into s->buf; returns the count,
 * or -1 on allocation failure. */
static int64_t row_partners(const bk_t *h, scratch_t *s, int64_t i, int sorted) {
    const int64_t nw = h->nwords;
    const uint64_t *wi = h->wloc + i * nw;
    int64_t m = 0;
    uint32_t maxj = 0;
    s->stamp[i] = (int32_t)i; /* no self pair */
    for (int64_t e = h->roff[i]; e < h->roff[i + 1]; ++e) {
        int32_t c = h->rcolors[e];
        for (int64_t t = h->bstart[c]; t < h->bstart[c + 1]; ++t) {
            int32_t j = h->bmem[t];
            if (s->stamp[j] == (int32_t)i) continue;
            s->stamp[j] = (int32_t)i;
            if (anticommute(wi, h->wloc + (int64_t)j * nw, nw)) continue;
            if (m == s->cap) {
                int64_t nc = 2 * s->cap;
                uint32_t *nb = (uint32_t *)realloc(s->buf, (size_t)nc * sizeof(uint32_t));
                if (!nb) return -1;
                s->buf = nb;
                uint32_t *nt = (uint32_t *)realloc(s->tmp, (size_t)nc * sizeof(uint32_t));
                if (!nt) return -1;
                s->tmp = nt;
                s->cap = nc;
            }
            s->buf[m++] = (uint32_t)j;
            if ((uint32_t)j > maxj) maxj = (uint32_t)j;
        }
    }
    if (sorted && m > 1) radix_sort_u32(s->buf, s->tmp, m, maxj);
    return m;
}

/* Degrees (both directions) of local rows [lo, hi) and, optionally, the upper degrees
 * (partners j > i; the one-phase budget projection).  Returns 0 or -1. */
int bk_degrees(const bk_t *h, int64_t lo, int64_t hi, int64_t *deg, int64_t *deg_upper) {
    scratch_t s;
    if (scratch_init(&s, h)) {
        scratch_free(&s);
        return -1;
    }
    int rc = 0;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t m = row_partners(h, &s, i, 0);
        if (m < 0) {
            rc = -1;
            break;
        }
        deg[i - lo] = m;
        if (deg_upper) {
            int64_t u = 0;
            for (int64_t k = 0; k < m; ++k) u += s.buf[k] > (uint32_t)i;
            deg_upper[i - lo] = u;
        }
    }
    scratch_free(&s);
    return rc;
}

/* The sorted conflict rows of local rows [lo, hi), concatenated into out (int64): compact
 * ids when a compaction map is set, local ids otherwise.  Returns the entries written or
 * -1.  The caller sizes out from bk_degrees. */
int64_t bk_emit(const bk_t *h, int64_t lo, int64_t hi, int64_t *out) {
    scratch_t s;
    if (scratch_init(&s, h)) {
        scratch_free(&s);
        return -1;
    }
    int64_t w = 0;
    for (int64_t i = lo; i < hi; ++i) {
        int64_t m = row_partners(h, &s, i, 1);
        if (m < 0) {
            w = -1;
            break;
        }
        if (h->cid)
            for (int64_t k = 0; k < m; ++k) out[w + k] = h->cid[s.buf[k]];
        else
            for (int64_t k = 0; k < m; ++k) out[w + k] = (int64_t)s.buf[k];
        w += m;
    }
    scratch_free(&s);
    return w;
}

/* ---- view_edges_scanned: commuting pairs i < j, for i in [lo, hi) ------------------------
 * The words are transposed to one array per word (structure of arrays) and the pair space is
 * walked in row blocks x column tiles, so a tile stays in cache for a block of rows. */
typedef struct {
    const bk_t *h;
    uint64_t *soa;           /* (nwords, n) */
    int64_t lo, hi, next;
    int64_t total;
    pthread_mutex_t lock;
} cc_job_t;

#define CC_ROWS 64
#define CC_TILE 4096

static void *cc_worker(void *arg) {
    cc_job_t *jb = (cc_job_t *)arg;
    const int64_t n = jb->h->n, nw = jb->h->nwords;
    int64_t mine = 0;
    for (;;) {
        pthread_mutex_lock(&jb->lock);
        int64_t r0 = jb->next;
        jb->next += CC_ROWS;
        pthread_mutex_unlock(&jb->lock);
        if (r0 >= jb->hi) break;
        int64_t r1 = r0 + CC_ROWS < jb->hi ? r0 + CC_ROWS : jb->hi;
        for (int64_t t0 = r0 + 1; t0 < n; t0 += CC_TILE) {
            int64_t t1 = t0 + CC_TILE < n ? t0 + CC_TILE : n;
            for (int64_t i = r0; i < r1; ++i) {
                int64_t j0 = t0 > i + 1 ? t0 : i + 1;
                if (j0 >= t1) continue;
                int64_t odd = 0;
                if (nw == 1) {
                    const uint64_t a0 = jb->h->wloc[i];
                    const uint64_t *c0 = jb->soa;
                    for (int64_t j = j0; j < t1; ++j) odd += __builtin_popcountll(c0[j] & a0) & 1;
                } else if (nw == 2) {
                    const uint64_t a0 = jb->h->wloc[2 * i], a1 = jb->h->wloc[2 * i + 1];
                    const uint64_t *c0 = jb->soa, *c1 = jb->soa + n;
                    for (int64_t j = j0; j < t1; ++j)
                        odd += __builtin_popcountll((c0[j] & a0) ^ (c1[j] & a1)) & 1;
                } else if (nw == 3) {
                    const uint64_t *a = jb->h->wloc + 3 * i;
                    const uint64_t a0 = a[0], a1 = a[1], a2 = a[2];
                    const uint64_t *c0 = jb->soa, *c1 = jb->soa + n, *c2 = jb->soa + 2 * n;
                    for (int64_t j = j0; j < t1; ++j)
                        odd += __builtin_popcountll((c0[j] & a0) ^ (c1[j] & a1) ^ (c2[j] & a2)) & 1;
                } else {
                    const uint64_t *a = jb->h->wloc + nw * i;
                    for (int64_t j = j0; j < t1; ++j) {
                        uint64_t acc = 0;
                        for (int64_t w = 0; w < nw; ++w) acc ^= jb->soa[w * n + j] & a[w];
                        odd += __builtin_popcountll(acc) & 1;
                    }
                }
                mine += (t1 - j0) - odd;
            }
        }
    }
    pthread_mutex_lock(&jb->lock);
    jb->total += mine;
    pthread_mutex_unlock(&jb->lock);
    return NULL;
}

int64_t bk_commute_count(const bk_t *h, int64_t lo, int64_t hi, int threads) {
    const int64_t n = h->n, nw = h->nwords;
    if (n < 2) return 0;
    cc_job_t jb;
    memset(&jb, 0, sizeof jb);
    jb.h = h;
    jb.soa = (uint64_t *)malloc((size_t)n * (size_t)nw * sizeof(uint64_t));
    if (!jb.soa) return -1;
    for (int64_t k = 0; k < n; ++k)
        for (int64_t w = 0; w < nw; ++w) jb.soa[w * n + k] = h->wloc[k * nw + w];
    jb.lo = lo;
    jb.hi = hi < n ? hi : n;
    jb.next = lo;
    pthread_mutex_init(&jb.lock, NULL);
    if (threads < 1) threads = 1;
    if (threads > 256) threads = 256;
    pthread_t tid[256];
    for (int t = 1; t < threads; ++t) pthread_create(&tid[t], NULL, cc_worker, &jb);
    cc_worker(&jb);
    for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
    pthread_mutex_destroy(&jb.lock);
    free(jb.soa);
    return jb.total;
}

int64_t bk_n(const bk_t *h) { return h->n; }
