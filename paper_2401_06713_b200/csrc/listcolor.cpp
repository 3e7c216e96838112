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
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
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
int pcg_color_dynamic(int64_t nm, const int64_t *offsets, const int64_t *neighbors,
                      const int64_t *list_data, const int64_t *list_off, uint64_t *rng6,
                      int64_t *color_of, int64_t *removal_ops) {
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
    int32_t top = 0;
    for (int64_t k = 0; k < nm; ++k) {
        const int64_t l = list_off[k + 1] - list_off[k];
        if (l > INT32_MAX) return -1;
        len[k] = (int32_t)l;
        top = std::max(top, len[k]);
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
        for (int64_t e = offsets[v]; e < offsets[v + 1]; ++e) {
            const int32_t u = (int32_t)neighbors[e];
            if (done[u]) continue;
            int64_t *ur = cols.data() + list_off[u];
            int32_t pos = -1;
            for (int32_t x = 0; x < len[u]; ++x)
                if (ur[x] == c) {
                    pos = x;
                    break;
                }
            if (pos < 0) continue;
            ++removals;
            ur[pos] = ur[len[u] - 1];  // swap-with-last (the Python dict keeps positions in sync)
            --len[u];
            unlink(u);
            if (len[u] == 0) {
                done[u] = 1;
                --left;
                continue;
            }
            const int32_t b = len[u];
            bucket_of[u] = b;
            slot_of[u] = (int32_t)buckets[b].size();
            buckets[b].push_back(u);
            if (b < lowest) lowest = b;
        }
    }
    *removal_ops = removals;
    // hand the advanced generator state back (numpy's Generator continues from here)
    rng6[0] = (uint64_t)(g.state >> 64);
    rng6[1] = (uint64_t)g.state;
    rng6[4] = g.has32 ? 1u : 0u;
    rng6[5] = g.half;
    return 0;
}

}  // extern "C"
