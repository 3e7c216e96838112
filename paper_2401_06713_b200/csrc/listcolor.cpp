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
#include <atomic>
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
 * removals, bucket moves and draws are the sequential ones.  A 64-bit color signature per
 * member (bit c & 63 of each listed color) skips most list scans.
 */
int pcg_color_dynamic_mt(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                         const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                         int64_t *color_of, int64_t *removal_ops, int32_t threads,
                         int64_t par_min_deg) {
    Pcg64 g;
    g.state = ((unsigned __int128)rng6[0] << 64) | rng6[1];
    g.inc = ((unsigned __int128)rng6[2] << 64) | rng6[3];
    g.has32 = rng6[4] != 0;
    g.half = (uint32_t)rng6[5];
    *removal_ops = 0;
    if (nm == 0) return 0;

    // per-member mutable lists (value + position map via linear search: lists are short)
    std::vector<int64_t> cols(list_data, list_data + list_off[nm]);
    std::vector<int32_t> len(nm);
    std::vector<uint64_t> sig(nm, 0);
    int32_t top = 0;
    for (int64_t k = 0; k < nm; ++k) {
        const int64_t l = list_off[k + 1] - list_off[k];
        if (l > INT32_MAX) return -1;
        len[k] = (int32_t)l;
        top = std::max(top, len[k]);
        for (int64_t x = list_off[k]; x < list_off[k + 1]; ++x) sig[k] |= 1ull << (cols[x] & 63);
    }
    std::vector<std::vector<int32_t>> buckets(top + 1);
    std::vector<int32_t> bucket_of(nm), slot_of(nm);
    for (int64_t k = 0; k < nm; ++k) {
        const int32_t b = len[k];
        bucket_of[k] = b;
        slot_of[k] = (int32_t)buckets[b].size();
        buckets[b].push_back((int32_t)k);
    }
    std::vector<uint8_t> done(nm, 0);
    for (int64_t k = 0; k < nm; ++k) color_of[k] = INT64_MIN;
    int64_t left = nm, removals = 0;
    int32_t lowest = 0;
    auto unlink = [&](int32_t k) {
        std::vector<int32_t> &bk = buckets[bucket_of[k]];
        const int32_t s = slot_of[k];
        const int32_t tail = bk.back();
        bk[s] = tail;
        slot_of[tail] = s;
        bk.pop_back();
    };
    // position of color c in u's list, or -1 (signature first)
    auto find = [&](int32_t u, int64_t c) -> int32_t {
        if (!((sig[u] >> (c & 63)) & 1u)) return -1;
        const int64_t *ur = cols.data() + list_off[u];
        for (int32_t x = 0; x < len[u]; ++x)
            if (ur[x] == c) return x;
        return -1;
    };
    auto apply = [&](int32_t u, int32_t pos) {
        ++removals;
        int64_t *ur = cols.data() + list_off[u];
        ur[pos] = ur[len[u] - 1];  // swap-with-last (the Python dict keeps positions in sync)
        --len[u];
        uint64_t sg = 0;
        for (int32_t x = 0; x < len[u]; ++x) sg |= 1ull << (ur[x] & 63);
        sig[u] = sg;
        unlink(u);
        if (len[u] == 0) {
            done[u] = 1;
            --left;
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
    int64_t job_e0 = 0, job_e1 = 0, job_c = 0;
    auto scan = [&](int t) {
        const int64_t span = job_e1 - job_e0;
        const int64_t a = job_e0 + span * t / W, b = job_e0 + span * (t + 1) / W;
        auto &h = hits[t];
        h.clear();
        for (int64_t e = a; e < b; ++e) {
            const int32_t u = (int32_t)neighbors[e];
            if (done[u]) continue;
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
        done[v] = 1;
        --left;
        int64_t *row = cols.data() + list_off[v];
        const int64_t c = row[g.below((uint64_t)len[v])];
        color_of[v] = c;
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
                if (done[u]) continue;
                const int32_t pos = find(u, c);
                if (pos >= 0) apply(u, pos);
            }
        }
    }
    stop.store(true);
    for (auto &t : pool) t.join();
    *removal_ops = removals;
    // hand the advanced generator state back (numpy's Generator continues from here)
    rng6[0] = (uint64_t)(g.state >> 64);
    rng6[1] = (uint64_t)g.state;
    rng6[4] = g.has32 ? 1u : 0u;
    rng6[5] = g.half;
    return 0;
}

}  // extern "C"
