// Host list coloring of the conflict graph (Algorithm 2, dynamic bucket scheme) — a native
// port of palettecolor.list_coloring.color_dynamic (list_coloring.py:53-139) that makes the
// same random draws in the same order, so the coloring is bit-identical.
//
// Random stream: numpy's Generator(PCG64) — 128-bit LCG, XSL-RR 64-bit output, 32-bit draws
// served from the upper/lower halves of one 64-bit output (has_uint32 buffer), and
// Generator.integers(k) = Lemire's bounded rejection on 32-bit draws for k <= 2^32 (no draw
// at all for k == 1).  The caller passes the generator state numpy itself derived from
// SeedSequence([seed & (2^63-1), iteration, 0xC01]) (list_coloring.py:230), so seeding is
// exact by construction.
#include <immintrin.h>

#include <algorithm>
#include <type_traits>
#include <atomic>
#include <new>
#include <sys/mman.h>
#include <cstdio>
#include <cstdlib>
#include <climits>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Pcg64 {
    unsigned __int128 state, inc;
    bool has32 = false;
    uint32_t half = 0;

    static constexpr unsigned __int128 MULT =
        ((unsigned __int128)2549297995355413924ULL << 64) | 4865540595714422341ULL;

    uint64_t next64() {
        state = state * MULT + inc;
        const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        const uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64 - rot) & 63));
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return half;
        }
        const uint64_t v = next64();
        has32 = true;
        half = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // Generator.integers(k) for 1 <= k <= 2^32 (int64 dtype, endpoint=False)
    uint32_t below(uint64_t k) {
        if (k <= 1) return 0;  // rng == 0: numpy returns without drawing
        const uint32_t rng = (uint32_t)(k - 1);
        const uint64_t excl = (uint64_t)rng + 1;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t thr = (uint32_t)((UINT32_MAX - rng) % excl);
            while (left < thr) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return (uint32_t)(m >> 32);
    }
};

// A flat array on 2 MB pages (madvise: the box's THP mode).  The coloring's arrays are
// 0.1-0.3 GB each at config 3 and are read at random: on 4 KB pages most of those reads also
// miss the TLB.
template <typename T>
struct HBuf {
    T *p = nullptr;
    size_t n = 0;
    explicit HBuf(size_t count) : n(count) {
        const size_t H = (size_t)2 << 20;
        const size_t bytes = ((std::max<size_t>(count * sizeof(T), 1) + H - 1) / H) * H;
        p = static_cast<T *>(std::aligned_alloc(H, bytes));
        if (!p) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);
    }
    HBuf(size_t count, T v) : HBuf(count) { std::fill(p, p + n, v); }
    ~HBuf() { std::free(p); }
    HBuf(const HBuf &) = delete;
    HBuf &operator=(const HBuf &) = delete;
    T &operator[](size_t i) { return p[i]; }
    const T &operator[](size_t i) const { return p[i]; }
    T *data() { return p; }
    size_t size() const { return n; }
};

// One size bucket of the dynamic scheme's queue, a slice of one big array on huge pages
// (a bucket never holds more than nm members); the std::vector operations the queue uses.
struct FlatBucket {
    int32_t *p = nullptr;
    int32_t n = 0;
    bool empty() const { return n == 0; }
    size_t size() const { return (size_t)n; }
    int32_t &operator[](size_t i) { return p[i]; }
    int32_t back() const { return p[n - 1]; }
    void pop_back() { --n; }
    void push_back(int32_t v) { p[n++] = v; }
    int32_t *data() { return p; }
};

}  // namespace

extern "C" {

/*
 * nm members; CSR (offsets nm+1, neighbors) over compact ids; member k's color list is
 * list_data[list_off[k] .. list_off[k+1]) in the caller's order (ColorLists row order).
 * rng6: {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger} of numpy's PCG64, updated
 * in place to the state after the last draw.
 * Outputs: color_of[k] (color, or INT64_MIN for the residue), *removal_ops.
 * Returns 0, or -1 on a list longer than 2^31.
 */
int pcg_color_dynamic_mt(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                         const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                         int64_t *color_of, int64_t *removal_ops, int32_t threads,
                         int64_t par_min_deg);

int pcg_color_dynamic(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                      const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                      int64_t *color_of, int64_t *removal_ops) {
    return pcg_color_dynamic_mt(nm, offsets, neighbors, list_data, list_off, rng6, color_of,
                                removal_ops, 0, -1);
}

/*
 * Same coloring, with the neighbor scan of each step split across `threads` host threads
 * (0: up to 16) when the picked member has at least `par_min_deg` neighbors (-1: 512).
 * A step only reads the neighbors' lists to find the picked color (a neighbor's list changes
 * only through its own removal, and a row lists each neighbor once), so the threads scan
 * contiguous slices of the row and the calling thread applies the hits in row order: the
 * removals, bucket moves and draws are the sequential ones.
 *
 * The scan's filter is a 256-bit color signature per member (bit c & 255 of every listed
 * color; a finished member's signature is zeroed, so it also stands for `processed`): one
 * random 8-byte load per neighbor, and a list scan only on a signature hit (~10% of the
 * neighbors at 28 colors per list).  A removal leaves the signature as it is — a stale bit
 * only costs a list scan that finds nothing, so the filter stays exact.  Colors are held as
 * int32 when the palette allows (half the bytes per list scan).
 */
}  // extern "C"

namespace {

template <typename C>
int color_dynamic_impl(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                       const int64_t *list_data, const int64_t *list_off, Pcg64 &g,
                       int64_t *color_of, int64_t *removal_ops, int32_t threads,
                       int64_t par_min_deg) {
    std::vector<C> cols(list_off[nm]);
    for (int64_t x = 0; x < list_off[nm]; ++x) cols[x] = (C)list_data[x];
    std::vector<int32_t> len(nm);
    std::vector<uint64_t> sig((size_t)nm * 4, 0);
    int32_t top = 0;
    for (int64_t k = 0; k < nm; ++k) {
        const int64_t l = list_off[k + 1] - list_off[k];
        if (l > INT32_MAX) return -1;
        len[k] = (int32_t)l;
        top = std::max(top, len[k]);
        for (int64_t x = list_off[k]; x < list_off[k + 1]; ++x) {
            const uint64_t c = (uint64_t)cols[x];
            sig[4 * k + ((c >> 6) & 3)] |= 1ull << (c & 63);
        }
    }
    std::vector<std::vector<int32_t>> buckets(top + 1);
    std::vector<int32_t> bucket_of(nm), slot_of(nm);
    for (int64_t k = 0; k < nm; ++k) {
        const int32_t b = len[k];
        bucket_of[k] = b;
        slot_of[k] = (int32_t)buckets[b].size();
        buckets[b].push_back((int32_t)k);
    }
    for (int64_t k = 0; k < nm; ++k) color_of[k] = INT64_MIN;
    int64_t left = nm, removals = 0;
    int32_t lowest = 0;
    auto finish = [&](int32_t k) {  // colored or out of colors: never matched again
        uint64_t *sg = sig.data() + 4 * (size_t)k;
        sg[0] = sg[1] = sg[2] = sg[3] = 0;
        --left;
    };
    auto unlink = [&](int32_t k) {
        std::vector<int32_t> &bk = buckets[bucket_of[k]];
        const int32_t s = slot_of[k];
        const int32_t tail = bk.back();
        bk[s] = tail;
        slot_of[tail] = s;
        bk.pop_back();
    };
    // position of color c in u's list, or -1 (signature first)
    auto find = [&](int32_t u, C c) -> int32_t {
        const uint64_t cu = (uint64_t)c;
        if (!((sig[4 * (size_t)u + ((cu >> 6) & 3)] >> (cu & 63)) & 1u)) return -1;
        const C *ur = cols.data() + list_off[u];
        for (int32_t x = 0; x < len[u]; ++x)
            if (ur[x] == c) return x;
        return -1;
    };
    auto apply = [&](int32_t u, int32_t pos) {
        ++removals;
        C *ur = cols.data() + list_off[u];
        ur[pos] = ur[len[u] - 1];  // swap-with-last (the Python dict keeps positions in sync)
        --len[u];
        unlink(u);
        if (len[u] == 0) {
            finish(u);
            return;
        }
        const int32_t b = len[u];
        bucket_of[u] = b;
        slot_of[u] = (int32_t)buckets[b].size();
        buckets[b].push_back(u);
        if (b < lowest) lowest = b;
    };

    // worker pool for the wide steps
    const int64_t nnz = offsets[nm] - offsets[0];
    int W = threads > 0 ? threads : (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    const int64_t pmin = par_min_deg >= 0 ? par_min_deg : 512;
    if (nnz < (int64_t)1 << 20 && threads <= 0) W = 1;  // small graphs: not worth the threads
    std::vector<std::vector<std::pair<int32_t, int32_t>>> hits(W);
    std::atomic<uint64_t> epoch{0};
    std::atomic<int> pending{0};
    std::atomic<bool> stop{false};
    int64_t job_e0 = 0, job_e1 = 0;
    C job_c = 0;
    auto scan = [&](int t) {
        const int64_t span = job_e1 - job_e0;
        const int64_t a = job_e0 + span * t / W, b = job_e0 + span * (t + 1) / W;
        auto &h = hits[t];
        h.clear();
        for (int64_t e = a; e < b; ++e) {
            const int32_t u = (int32_t)neighbors[e];
            const int32_t pos = find(u, job_c);
            if (pos >= 0) h.emplace_back(u, pos);
        }
    };
    std::vector<std::thread> pool;
    for (int t = 1; t < W; ++t)
        pool.emplace_back([&, t] {
            uint64_t seen = 0;
            for (;;) {
                uint64_t ep;
                while ((ep = epoch.load(std::memory_order_acquire)) == seen) {
                    if (stop.load(std::memory_order_relaxed)) return;
                    _mm_pause();
                }
                seen = ep;
                scan(t);
                pending.fetch_sub(1, std::memory_order_release);
            }
        });

    while (left) {
        while (buckets[lowest].empty()) ++lowest;
        std::vector<int32_t> &bk = buckets[lowest];
        const int32_t v = bk[g.below(bk.size())];
        unlink(v);
        finish(v);
        C *row = cols.data() + list_off[v];
        const C c = row[g.below((uint64_t)len[v])];
        color_of[v] = (int64_t)c;
        const int64_t e0 = offsets[v], e1 = offsets[v + 1];
        if (W > 1 && e1 - e0 >= pmin) {
            job_e0 = e0;
            job_e1 = e1;
            job_c = c;
            pending.store(W - 1, std::memory_order_relaxed);
            epoch.fetch_add(1, std::memory_order_release);
            scan(0);
            while (pending.load(std::memory_order_acquire) != 0) _mm_pause();
            for (int t = 0; t < W; ++t)
                for (const auto &h : hits[t]) apply(h.first, h.second);
        } else {
            for (int64_t e = e0; e < e1; ++e) {
                const int32_t u = (int32_t)neighbors[e];
                const int32_t pos = find(u, c);
                if (pos >= 0) apply(u, pos);
            }
        }
    }
    stop.store(true);
    for (auto &t : pool) t.join();
    *removal_ops = removals;
    return 0;
}

// The same coloring driven by color buckets instead of neighbor scans.  A step colors v with
// c and must strike c from every unprocessed neighbor u that still lists c, in row order.
// Those u are exactly the live members of c's color bucket (members listing c, ascending,
// not yet processed, c not yet struck) that are neighbors of v — so the step walks c's bucket
// (~m = n L / P entries, each bucket walked once per vertex colored c) and tests adjacency by
// galloping through v's sorted row, instead of touching all deg(v) neighbors.  At config 3:
// ~2e8 bucket entries over the run instead of 3.1e9 neighbor visits, single-threaded.  The
// hits come out ascending (the row order), so removals, bucket moves and draws are the
// sequential ones.  Each list position carries its bucket entry (moved along with the color
// on swap-with-last), each entry its live flag and current list position.  Returns 1 when
// the colors do not fit (range > 2^28) or a list repeats a color: the caller takes the scan.
template <typename C, typename Adjacent>
int color_dynamic_buckets(int64_t nm, Adjacent &&adjacent, const int64_t *list_data,
                          const int64_t *list_off, Pcg64 &g, int64_t *color_of,
                          int64_t *removal_ops) {
    const int64_t tot = list_off[nm];
    int64_t cmin = INT64_MAX, cmax = INT64_MIN;
    for (int64_t x = 0; x < tot; ++x) {
        cmin = std::min(cmin, list_data[x]);
        cmax = std::max(cmax, list_data[x]);
    }
    if (tot == 0 || cmax - cmin >= ((int64_t)1 << 28)) return 1;
    const int64_t R = cmax - cmin + 1;
    // color buckets (counting sort by color, members ascending inside a bucket)
    std::vector<int64_t> bstart(R + 1, 0);
    for (int64_t x = 0; x < tot; ++x) ++bstart[list_data[x] - cmin + 1];
    for (int64_t r = 0; r < R; ++r) bstart[r + 1] += bstart[r];
    if (tot >= ((int64_t)1 << 31)) return 1;
    HBuf<int32_t> bmem(tot);
    HBuf<int32_t> ent(tot);      // list position -> its bucket entry
    HBuf<int32_t> eslot(tot);    // bucket entry -> its current list position
    HBuf<uint8_t> alive(tot, 1);
    {
        std::vector<int64_t> fillp(bstart.begin(), bstart.end() - 1);
        for (int64_t k = 0; k < nm; ++k)
            for (int64_t x = list_off[k]; x < list_off[k + 1]; ++x) {
                const int64_t r = list_data[x] - cmin;
                const int64_t p = fillp[r]++;
                if (p > bstart[r] && bmem[p - 1] == (int32_t)k) return 1;  // a repeated color
                bmem[p] = (int32_t)k;
                ent[x] = (int32_t)p;
                eslot[p] = (int32_t)(x - list_off[k]);
            }
    }
    HBuf<C> cols(tot);
    for (int64_t x = 0; x < tot; ++x) cols[x] = (C)list_data[x];
    // per member: remaining list length (= its size bucket while unprocessed) and its slot in
    // that bucket, side by side (one cache line per touched member)
    struct Mem {
        int32_t len, slot;
    };
    HBuf<Mem> ms(nm);
    int32_t top = 0;
    for (int64_t k = 0; k < nm; ++k) {
        ms[k].len = (int32_t)(list_off[k + 1] - list_off[k]);
        top = std::max(top, ms[k].len);
    }
    HBuf<int32_t> qdata((size_t)(top + 1) * (size_t)nm);
    std::vector<FlatBucket> buckets(top + 1);
    for (int32_t b = 0; b <= top; ++b) buckets[b].p = qdata.data() + (size_t)b * (size_t)nm;
    for (int64_t k = 0; k < nm; ++k) {
        FlatBucket &bk = buckets[ms[k].len];
        ms[k].slot = (int32_t)bk.size();
        bk.push_back((int32_t)k);
    }
    for (int64_t k = 0; k < nm; ++k) color_of[k] = INT64_MIN;
    int64_t left = nm, removals = 0;
    int32_t lowest = 0;
    std::vector<uint8_t> hit;     // batch tests of one bucket walk
    std::vector<int32_t> live;    // its live entries
    std::vector<int32_t> hits;    // positions of the hits in the walked bucket
    auto finish = [&](int32_t k) {  // processed: none of its remaining colors is live
        for (int64_t x = list_off[k]; x < list_off[k] + ms[k].len; ++x) alive[ent[x]] = 0;
        --left;
    };
    auto unlink = [&](int32_t k) {  // out of its size bucket (swap-with-last, as the reference)
        FlatBucket &bk = buckets[ms[k].len];
        const int32_t s = ms[k].slot;
        const int32_t tail = bk.back();
        bk[s] = tail;
        ms[tail].slot = s;
        bk.pop_back();
    };
    auto apply = [&](int32_t u, int64_t p) {  // strike entry p's color from u's list
        ++removals;
        alive[p] = 0;
        const int64_t base = list_off[u];
        const int32_t pos = eslot[p], last = ms[u].len - 1;
        cols[base + pos] = cols[base + last];  // swap-with-last, as the reference
        const int32_t el = ent[base + last];
        ent[base + pos] = el;
        eslot[el] = pos;
        unlink(u);  // from the bucket of its old size
        const int32_t b = --ms[u].len;
        if (b == 0) {
            --left;  // (no live entries left)
            return;
        }
        FlatBucket &nbk = buckets[b];
        ms[u].slot = (int32_t)nbk.size();
        nbk.push_back(u);
        if (b < lowest) lowest = b;
    };

    // PCG_TRACE_COLOR=1: cycle counts of the phases, printed to stderr (diagnostic)
    static const bool trace = getenv("PCG_TRACE_COLOR") != nullptr;
    uint64_t tc[4] = {0, 0, 0, 0}, scanned = 0;
    while (left) {
        const uint64_t a0 = trace ? __rdtsc() : 0;
        while (buckets[lowest].empty()) ++lowest;
        FlatBucket &bk = buckets[lowest];
        const int32_t v = bk[g.below(bk.size())];
        unlink(v);
        finish(v);
        const C *row = cols.data() + list_off[v];
        const C c = row[g.below((uint64_t)ms[v].len)];
        color_of[v] = (int64_t)c;
        // live members of c's bucket that are neighbors of v, ascending
        const int64_t rc = (int64_t)c - cmin;
        adjacent.start(v);
        if constexpr (std::decay_t<Adjacent>::kBatch) {
            // every live entry's test first, without branches (its loads overlap), then the
            // hits in order; an apply never changes another entry of the same bucket
            const int64_t b0 = bstart[rc], nb = bstart[rc + 1] - b0;
            if ((int64_t)hit.size() < nb) {
                hit.resize(nb);
                live.resize(nb);
            }
            const uint64_t a1 = trace ? __rdtsc() : 0;
            // the live entries (branch-free compaction), then their tests
            int32_t nl = 0;
            for (int64_t q = 0; q < nb; ++q) {
                live[nl] = (int32_t)q;
                nl += alive[b0 + q];
            }
            const uint64_t a15 = trace ? __rdtsc() : 0;
            if (trace) tc[3] += a15 - a1;
            constexpr int PF = 16;
            for (int32_t i = 0; i < nl; ++i) {
                if (i + PF < nl) adjacent.prefetch(bmem[b0 + live[i + PF]]);
                hit[i] = (uint8_t)adjacent.test(bmem[b0 + live[i]]);
            }
            hits.clear();
            for (int32_t i = 0; i < nl; ++i)
                if (hit[i]) hits.push_back(live[i]);
            const uint64_t a2 = trace ? __rdtsc() : 0;
            // the applies' scattered state is requested a few hits ahead: the member and its
            // list (distance 8), then its slot in its size bucket (distance 4)
            const int nh = (int)hits.size();
            for (int i = 0; i < nh; ++i) {
                if (i + 8 < nh) {
                    const int32_t w = bmem[b0 + hits[i + 8]];
                    __builtin_prefetch(&ms[w], 1);
                    __builtin_prefetch(cols.data() + list_off[w], 1);
                    __builtin_prefetch(ent.data() + list_off[w], 1);
                    __builtin_prefetch(&eslot[b0 + hits[i + 8]], 0);
                }
                if (i + 4 < nh) {
                    const int32_t w = bmem[b0 + hits[i + 4]];
                    __builtin_prefetch(buckets[ms[w].len].data() + ms[w].slot, 1);
                    // the entry of w's last listed color (its list position moves)
                    __builtin_prefetch(&eslot[ent[list_off[w] + ms[w].len - 1]], 1);
                }
                apply(bmem[b0 + hits[i]], b0 + hits[i]);
            }
            if (trace) {
                const uint64_t a3 = __rdtsc();
                tc[0] += a1 - a0;
                tc[1] += a2 - a1;
                tc[2] += a3 - a2;
                scanned += nl;
            }
        } else {
            for (int64_t p = bstart[rc]; p < bstart[rc + 1]; ++p) {
                if (!alive[p]) continue;
                const int r = adjacent.test(bmem[p]);
                if (r < 0) break;  // no neighbor beyond
                if (r) apply(bmem[p], p);
            }
        }
    }
    *removal_ops = removals;
    if (trace)
        fprintf(stderr, "color buckets: pick+finish %.3g, tests %.3g (live compaction %.3g), "
                "applies %.3g Gcycles; %lld live entries tested, %lld removals\n", tc[0] * 1e-9,
                tc[1] * 1e-9, tc[3] * 1e-9, tc[2] * 1e-9,
                (long long)scanned, (long long)removals);
    return 0;
}

// adjacency of the bucket members to the step's vertex: its sorted CSR row, galloping
// (members arrive ascending); test returns 1 adjacent, 0 not, -1 nothing adjacent beyond
struct RowAdjacency {
    static constexpr bool kBatch = false;
    const int64_t *offsets, *neighbors;
    const int64_t *nb = nullptr;
    int64_t deg = 0, r = 0;
    void start(int32_t v) {
        nb = neighbors + offsets[v];
        deg = offsets[v + 1] - offsets[v];
        r = 0;
    }
    void prefetch(int64_t) {}
    int test(int64_t u) {
        if (r >= deg) return -1;
        if (nb[r] < u) {  // gallop to the first row entry >= u
            int64_t step = 1;
            while (r + step < deg && nb[r + step] < u) step <<= 1;
            int64_t lo = r + (step >> 1) + 1, hi = std::min(deg, r + step);
            while (lo < hi) {
                const int64_t mid = (lo + hi) >> 1;
                if (nb[mid] < u) lo = mid + 1; else hi = mid;
            }
            r = lo;
            if (r >= deg) return -1;
        }
        return nb[r] == u ? 1 : 0;
    }
};

// adjacency from the Pauli words themselves (graph.py:327-336 implicit-complement mode): two
// members of a color bucket share that color, so they are conflict neighbors iff their
// strings commute — an even popcount of the ANDed 3-bit code words (pauli.py:258-268).  One
// independent 8*NW-byte load per tested member instead of a walk through the CSR row.
template <int NW>
struct WordAdjacency {
    static constexpr bool kBatch = true;
    const uint64_t *words;  // nm x nw, member order
    int nw;
    uint64_t wv[NW > 0 ? NW : 1];
    const uint64_t *pv = nullptr;
    void start(int32_t v) {
        pv = words + (size_t)v * nw;
        if (NW > 0)
            for (int k = 0; k < NW; ++k) wv[k] = pv[k];
    }
    void prefetch(int64_t u) { __builtin_prefetch(words + (size_t)u * nw); }
    int test(int64_t u) {
        const uint64_t *pu = words + (size_t)u * nw;
        uint64_t acc = 0;
        if (NW > 0) {
            for (int k = 0; k < NW; ++k) acc ^= pu[k] & wv[k];
        } else {
            for (int k = 0; k < nw; ++k) acc ^= pu[k] & pv[k];
        }
        return (int)((__builtin_popcountll(acc) & 1) ^ 1);
    }
};

template <typename Adj>
int buckets_any(bool fits32, int64_t nm, Adj &&adj, const int64_t *list_data,
                const int64_t *list_off, Pcg64 &g, int64_t *color_of, int64_t *removal_ops) {
    return fits32 ? color_dynamic_buckets<int32_t>(nm, adj, list_data, list_off, g, color_of, removal_ops)
                  : color_dynamic_buckets<int64_t>(nm, adj, list_data, list_off, g, color_of, removal_ops);
}

Pcg64 load_rng(const uint64_t *rng6) {
    Pcg64 g;
    g.state = ((unsigned __int128)rng6[0] << 64) | rng6[1];
    g.inc = ((unsigned __int128)rng6[2] << 64) | rng6[3];
    g.has32 = rng6[4] != 0;
    g.half = (uint32_t)rng6[5];
    return g;
}

void store_rng(const Pcg64 &g, uint64_t *rng6) {
    rng6[0] = (uint64_t)(g.state >> 64);
    rng6[1] = (uint64_t)g.state;
    rng6[4] = g.has32 ? 1u : 0u;
    rng6[5] = g.half;
}

bool colors_fit32(int64_t nm, const int64_t *list_data, const int64_t *list_off) {
    for (int64_t x = 0; x < list_off[nm]; ++x)
        if (list_data[x] < INT32_MIN || list_data[x] > INT32_MAX) return false;
    return true;
}

}  // namespace

extern "C" {

int pcg_color_dynamic_mt(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                         const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                         int64_t *color_of, int64_t *removal_ops, int32_t threads,
                         int64_t par_min_deg) try {
    Pcg64 g = load_rng(rng6);
    *removal_ops = 0;
    if (nm == 0) return 0;
    const bool fits32 = colors_fit32(nm, list_data, list_off);
    // color buckets (par_min_deg >= -1, the default) or the neighbor scan (par_min_deg < -1:
    // the threaded scan with |par_min_deg| - 2 as the threshold; also when buckets decline)
    int rc = 1;
    if (par_min_deg >= -1) {
        const Pcg64 g0 = g;
        rc = buckets_any(fits32, nm, RowAdjacency{offsets, neighbors}, list_data, list_off, g,
                         color_of, removal_ops);
        if (rc == 1) g = g0;  // declined before drawing
    } else {
        par_min_deg = -par_min_deg - 2;
    }
    if (rc == 1)
        rc = fits32 ? color_dynamic_impl<int32_t>(nm, offsets, neighbors, list_data, list_off, g,
                                                  color_of, removal_ops, threads, par_min_deg)
                    : color_dynamic_impl<int64_t>(nm, offsets, neighbors, list_data, list_off, g,
                                                  color_of, removal_ops, threads, par_min_deg);
    if (rc) return rc;
    store_rng(g, rng6);  // numpy's Generator continues from here
    return 0;
} catch (const std::bad_alloc &) {
    return -2;  // out of host memory (nothing escapes the C ABI)
}

/*
 * The same coloring for a conflict graph of a Pauli view, without its CSR: `words` are the
 * members' packed 3-bit code words (nm x nwords, member order: PauliSet.words[members]).
 * Returns 1 (nothing drawn) when the colors do not suit the bucket form (range > 2^28 or a
 * list repeating a color): the caller then runs pcg_color_dynamic_mt on the CSR.
 */
int pcg_color_dynamic_words(int64_t nm, const uint64_t *words, int32_t nwords,
                            const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                            int64_t *color_of, int64_t *removal_ops) try {
    Pcg64 g = load_rng(rng6);
    *removal_ops = 0;
    if (nm == 0) return 0;
    const bool fits32 = colors_fit32(nm, list_data, list_off);
    int rc;
    switch (nwords) {
        case 1: rc = buckets_any(fits32, nm, WordAdjacency<1>{words, 1, {}}, list_data, list_off, g, color_of, removal_ops); break;
        case 2: rc = buckets_any(fits32, nm, WordAdjacency<2>{words, 2, {}}, list_data, list_off, g, color_of, removal_ops); break;
        case 3: rc = buckets_any(fits32, nm, WordAdjacency<3>{words, 3, {}}, list_data, list_off, g, color_of, removal_ops); break;
        case 4: rc = buckets_any(fits32, nm, WordAdjacency<4>{words, 4, {}}, list_data, list_off, g, color_of, removal_ops); break;
        case 6: rc = buckets_any(fits32, nm, WordAdjacency<6>{words, 6, {}}, list_data, list_off, g, color_of, removal_ops); break;
        default: rc = buckets_any(fits32, nm, WordAdjacency<0>{words, nwords, {}}, list_data, list_off, g, color_of, removal_ops); break;
    }
    if (rc) return rc;
    store_rng(g, rng6);
    return 0;
} catch (const std::bad_alloc &) {
    return -2;
}

}  // extern "C"
