// Owned bucket masks (K2a) and the popcount count pass (K2c); the fills are in fillblk.cu / fill.cu / rows.cu.
//
// Ownership.  A conflict pair {u, v} is admitted through every color the two lists share;
// k_owned_masks keeps it only in the commute mask of the SMALLEST shared color.  Then each
// row's L mask rows are disjoint:
//   deg[i]  = sum over i's colors c of popc(mask_c[k_c(i)])       (no dedupe, no bitmap)
//   row i   = merge of L disjoint ascending runs                   (no duplicates)
// A pair {v_k, v_t} of bucket c shares a smaller color iff some c' < c lies in both lists.
// Per color, the CTA inserts (c', k) for every member k and every color c' < c of its list
// into a shared-memory hash table keyed by c'; a key met twice marks the pairs of its group as
// not owned by c, and their bits are cleared (a few per color: P(share >= 2 | share 1) is
// ~(L-1)^2/P).  Exact; colors whose hash would overflow make the build use the dedupe path.
#include <algorithm>
#include <climits>

#include "pcg_internal.cuh"

namespace pcg {

namespace {

constexpr int OWN_THREADS = 256;
constexpr int OWN_COLL = 2048;        // collision list capacity
constexpr int OWN_LCAP = 1024;        // direct ownership: default losers per level (o.lcap)
constexpr int OWN_BM_FILTER = 512;    // bitmap ownership: 16K-bit filter of the repeated colors
constexpr int OWN_BM_COLL = 1024;     // bitmap ownership: holders of the repeated colors

template <int KW>
struct Vec {
    uint32_t v[KW > 0 ? KW : 1];
    __device__ __forceinline__ void load(const uint32_t *A, int64_t i, int kw) {
#pragma unroll
        for (int k = 0; k < KW; ++k) v[k] = __ldg(A + i * KW + k);
    }
    __device__ __forceinline__ uint32_t parity(const uint32_t *B, int32_t j, int kw) const {
        uint32_t acc = 0;
        const uint32_t *b = B + (int64_t)j * KW;
#pragma unroll
        for (int k = 0; k < KW; ++k) acc ^= v[k] & __ldg(b + k);
        return __popc(acc) & 1u;
    }
};
template <>
struct Vec<0> {
    const uint32_t *a;
    __device__ __forceinline__ void load(const uint32_t *A, int64_t i, int kw) { a = A + i * kw; }
    __device__ __forceinline__ uint32_t parity(const uint32_t *B, int32_t j, int kw) const {
        uint32_t acc = 0;
        const uint32_t *b = B + (int64_t)j * kw;
        for (int k = 0; k < kw; ++k) acc ^= __ldg(a + k) & __ldg(b + k);
        return __popc(acc) & 1u;
    }
};

__device__ __forceinline__ uint32_t mix32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

// ---------------------------------------------------------------------------------------
// K2a (owned): one CTA per color.
// ---------------------------------------------------------------------------------------
template <int KW>
__global__ void __launch_bounds__(OWN_THREADS) k_owned_masks(BucketArgs b, OwnArgs o) {
    extern __shared__ __align__(16) uint32_t osm[];
    const int HS = o.hash_slots;
    uint32_t *table = osm;                                        // HS: (c'+1)<<12 | first k
    unsigned short *head = reinterpret_cast<unsigned short *>(osm + HS);  // HS: last coll + 1
    uint32_t *coll = osm + HS + HS / 2;                           // OWN_COLL: slot<<12 | k
    int32_t *link = reinterpret_cast<int32_t *>(coll + OWN_COLL); // OWN_COLL: previous in slot
    int32_t *sid = link + OWN_COLL;                               // member ids (m_cap)
    uint32_t *sB = reinterpret_cast<uint32_t *>(sid + o.m_cap);   // partner vectors (m_cap * kw)
    __shared__ int ncoll, overflow;
    const int tid = threadIdx.x;
    const int kw = b.kw;
    for (int x = tid; x < HS + HS / 2; x += OWN_THREADS) osm[x] = 0u;
    for (int64_t c = blockIdx.x; c < b.P; c += gridDim.x) {
        const int m = b.bstart[c + 1] - b.bstart[c];
        if (m < 2) {
            if (m == 1 && tid == 0) b.masks[b.maskoff[c]] = 0u;
            continue;
        }
        const int W = (m + 31) >> 5;
        const int32_t *mem = b.bmemp + b.bpos[c];
        uint32_t *out = b.masks + b.maskoff[c];
        if (tid == 0) {
            ncoll = 0;
            overflow = 0;
        }
        for (int t = tid; t < m; t += OWN_THREADS) sid[t] = mem[t];
        __syncthreads();
        for (int x = tid; x < m * kw; x += OWN_THREADS) sB[x] = __ldg(b.B + (int64_t)sid[x / kw] * kw + x % kw);
        __syncthreads();
        // ---- commute masks: thread k owns row k
        for (int k = tid; k < m; k += OWN_THREADS) {
            uint32_t av[KW > 0 ? KW : 16];
            for (int q = 0; q < kw; ++q) av[q] = __ldg(b.A + (int64_t)sid[k] * kw + q);
            for (int w = 0; w < W; ++w) {
                uint32_t bits = 0u;
                const int tend = min(32, m - 32 * w);
                for (int tt = 0; tt < tend; ++tt) {
                    const uint32_t *bt = sB + (32 * w + tt) * kw;
                    uint32_t acc = 0u;
                    if constexpr (KW > 0) {
#pragma unroll
                        for (int q = 0; q < KW; ++q) acc ^= av[q] & bt[q];
                    } else {
                        for (int q = 0; q < kw; ++q) acc ^= av[q] & bt[q];
                    }
                    bits |= ((__popc(acc) & 1u) ^ 1u) << tt;
                }
                if (k >> 5 == w) bits &= ~(1u << (k & 31));  // no self pair
                out[(int64_t)k * W + w] = bits;
            }
        }
        // ---- ownership: (c', k) for every color c' < c of every member's list.  The first
        // holder of c' stays in the table; later ones go to the collision list, chained per
        // slot, so every pair of a group is produced exactly once (by its later member).
        for (int k = tid; k < m; k += OWN_THREADS) {
            const int32_t r = sid[k];
            const int64_t lo = o.loff ? o.loff[r] : (int64_t)r * o.L;
            const int64_t hi = o.loff ? o.loff[r + 1] : lo + o.L;
            for (int64_t x = lo; x < hi; ++x) {
                const int32_t cx = o.lrel[x];
                if (cx >= c) continue;
                const uint32_t cp = (uint32_t)cx + 1u;
                const uint32_t key = (cp << 12) | (uint32_t)k;
                uint32_t slot = mix32(cp) & (HS - 1);
                for (int probe = 0;; ++probe) {
                    if (probe == HS) {
                        overflow = 1;
                        break;
                    }
                    const uint32_t prev = atomicCAS(&table[slot], 0u, key);
                    if (prev == 0u) break;
                    if ((prev >> 12) == cp) {
                        const int q = atomicAdd(&ncoll, 1);
                        if (q < OWN_COLL) {
                            coll[q] = (slot << 12) | (uint32_t)k;
                            // 16-bit chain head: swap through the containing 32-bit word
                            uint32_t *hw = reinterpret_cast<uint32_t *>(head) + (slot >> 1);
                            const int sh = (slot & 1) * 16;
                            uint32_t old = *hw, assumed;
                            do {
                                assumed = old;
                                const uint32_t nv = (assumed & ~(0xffffu << sh)) | ((uint32_t)(q + 1) << sh);
                                old = atomicCAS(hw, assumed, nv);
                            } while (old != assumed);
                            link[q] = (int)((old >> sh) & 0xffffu) - 1;
                        } else {
                            overflow = 1;
                        }
                        break;
                    }
                    slot = (slot + 1) & (HS - 1);
                }
            }
        }
        __syncthreads();
        const int nc = min(ncoll, OWN_COLL);
        if (overflow && tid == 0) atomicMax(o.overflow, overflow);
        for (int q = tid; q < nc; q += OWN_THREADS) {
            const uint32_t slot = coll[q] >> 12;
            const int k2 = (int)(coll[q] & 0xfffu);
            int k1 = (int)(table[slot] & 0xfffu);
            for (int p = link[q];; p = link[p]) {
                if (k1 != k2) {
                    atomicAnd(&out[(int64_t)k1 * W + (k2 >> 5)], ~(1u << (k2 & 31)));
                    atomicAnd(&out[(int64_t)k2 * W + (k1 >> 5)], ~(1u << (k1 & 31)));
                }
                if (p < 0) break;
                k1 = (int)(coll[p] & 0xfffu);
            }
        }
        __syncthreads();
        // reset the table and the chain heads this color touched
        for (int x = 4 * tid; x < HS; x += 4 * OWN_THREADS)
            *reinterpret_cast<uint4 *>(table + x) = make_uint4(0u, 0u, 0u, 0u);
        for (int q = tid; q < nc; q += OWN_THREADS) head[coll[q] >> 12] = 0;  // (16-bit store)
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// K2a (owned, four-Russians): one CTA per color, same output as k_owned_masks.  The m x m
// commute matrix of a bucket is a GF(2) product A_k . B_t: for each 32-partner word w the
// CTA transposes the partners' bits with ballots (BT[p] bit tt = bit p of B_{32w+tt}) and
// tabulates, for every 4-bit slice g of the K = 32*KW bits, the 16 XOR-combinations of
// BT[4g..4g+3].  Row k's mask word is then the XOR of NIB = 8*KW table entries picked by its
// own nibbles (addresses precomputed once per color): 32 pairs per NIB LDS + NIB/2 LOP3,
// instead of one AND/POPC chain per pair.  Ownership inserts run warp-per-member with the
// lanes over the member's (sorted) list, colors below c only.
// ---------------------------------------------------------------------------------------
template <int KW, bool DB>
__global__ void __launch_bounds__(OWN_THREADS, (KW <= 4 ? 4 : 3)) k_owned_fr(BucketArgs b, OwnArgs o) {
    constexpr int NIB = 8 * KW;
    extern __shared__ __align__(16) uint32_t osm[];
    const int HS = o.hash_slots;
    // ownership state: hash (large palettes) or a direct-mapped table over the colors
    uint32_t *table = osm;                                        // HS: (c'+1)<<12 | first k
    uint32_t *coll = osm + HS;                                    // OWN_COLL: slot<<12 | k
    unsigned short *dtab = reinterpret_cast<unsigned short *>(osm);  // direct: P member tags
    uint32_t *lA = osm + o.dtab_words;                            // direct: losers (c'<<12|k)
    const int lcap = o.lcap > 0 ? o.lcap : OWN_LCAP;
    uint32_t *lB = lA + lcap;
    // bitmap mode: bit c' of bm = color c' < c seen in the bucket; filt = a 16K-bit hash
    // filter of the colors seen twice; coll = their holders (c'<<12 | k), the filter's false
    // positives included (they pair with nothing: the pairing compares the colors)
    uint32_t *bm = osm, *filt = osm + o.bm_words;
    if (o.bitmap) coll = osm + o.bm_words + OWN_BM_FILTER;
    const int coll_cap = o.bitmap ? OWN_BM_COLL : OWN_COLL;
    const int state_words = o.bitmap ? o.bm_words + OWN_BM_FILTER : HS;  // zeroed per color
    int32_t *sid = reinterpret_cast<int32_t *>(
        osm + (o.direct ? o.dtab_words + 2 * lcap
                        : o.bitmap ? o.bm_words + OWN_BM_FILTER + OWN_BM_COLL : HS + OWN_COLL));
    constexpr int NB = DB ? 2 : 1;  // table buffers
    uint32_t *T = reinterpret_cast<uint32_t *>(sid + ((o.m_cap + 3) & ~3));  // NB x NIB*16 tables
    uint32_t *BT = T + NB * NIB * 16;                             // NB x 32*KW transposed bits
    uint32_t *sB = BT + NB * 32 * KW;                             // partner vectors, stride KW+1
    // row stride: odd (conflict-free transposition loads) from KW = 4; at KW = 2 the 2-way
    // conflict is cheaper than the padding (which would cost a CTA per SM at config 2)
    constexpr int SBS = KW >= 4 ? KW + 1 : KW;
    // members' color lists (rectangular lists): u16 when the palette allows, else u32
    void *sLv = sB + ((o.m_cap * SBS + 3) & ~3);
    unsigned short *sL16 = reinterpret_cast<unsigned short *>(sLv);
    int32_t *sL32 = reinterpret_cast<int32_t *>(sLv);
    const bool stage_lists = o.stage_lists != 0;
    __shared__ int ncoll, overflow, nlose, nlo, nhi;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int NWARPS = OWN_THREADS / 32;
    const uint32_t T_s = (uint32_t)__cvta_generic_to_shared(T);
    if (o.direct) {
        for (int x = tid; x < o.dtab_words; x += OWN_THREADS) osm[x] = 0u;
    } else {
        for (int x = tid; x < state_words; x += OWN_THREADS) osm[x] = 0u;
    }
    __shared__ long long witem;
    for (int64_t c = work_first(o.work, &witem); c < b.P; c = work_next(o.work, &witem, c)) {
        const int m = b.bstart[c + 1] - b.bstart[c];
        if (m < 2) {
            if (m == 1 && tid == 0) b.masks[b.maskoff[c]] = 0u;
            continue;
        }
        const int W = (m + 31) >> 5;
        const int32_t *mem = b.bmemp + b.bpos[c];
        uint32_t *out = b.masks + b.maskoff[c];
        if (tid == 0) {
            ncoll = 0;
            overflow = 0;
        }
        if (tid == 0) {
            nlo = 0;
            nhi = 0;
        }
        __syncthreads();
        {
            int lo_c = 0, hi_c = 0;
            for (int t = tid; t < m; t += OWN_THREADS) {
                const int32_t r = mem[t];
                sid[t] = r;
                lo_c += r < o.row_lo;
                hi_c += r < o.row_hi;
            }
            if (lo_c) atomicAdd(&nlo, lo_c);
            if (hi_c) atomicAdd(&nhi, hi_c);
        }
        __syncthreads();
        // members are ascending: this shard's mask rows are the positions [nlo, nhi)
        const int k_lo = nlo, k_hi = nhi;
        // stage the members' partner vectors and color lists once (all loads in flight
        // together; every later pass reads shared memory)
        for (int x = tid; x < m * KW; x += OWN_THREADS)
            sB[(x / KW) * SBS + x % KW] = __ldg(b.B + (int64_t)sid[x / KW] * KW + x % KW);
        if (stage_lists) {
            const uint32_t items = (uint32_t)m * (uint32_t)o.L;
            for (uint32_t e = tid; e < items; e += OWN_THREADS) {
                const int k = (int)__umulhi(e, o.l_magic);
                const int32_t cx = __ldg(o.lrel + (int64_t)sid[k] * o.L + (e - (uint32_t)k * (uint32_t)o.L));
                if (o.l16) sL16[e] = (unsigned short)cx; else sL32[e] = cx;
            }
        }
        __syncthreads();
        // ---- commute masks (rows of this shard's members only)
        for (int k0 = k_lo; k0 < k_hi; k0 += OWN_THREADS) {
            const int k = k0 + tid < k_hi ? k0 + tid : m;  // m: no row
            uint32_t naddr[NIB];
            {
                uint32_t av[KW];
                if (k < m) {  // the row's bits in 16-byte loads (one request per row)
                    const uint32_t *ar = b.A + (int64_t)sid[k] * KW;
                    if constexpr (KW % 4 == 0) {
#pragma unroll
                        for (int q = 0; q < KW; q += 4) {
                            const uint4 t4 = __ldg(reinterpret_cast<const uint4 *>(ar + q));
                            av[q] = t4.x; av[q + 1] = t4.y; av[q + 2] = t4.z; av[q + 3] = t4.w;
                        }
                    } else if constexpr (KW % 2 == 0) {
#pragma unroll
                        for (int q = 0; q < KW; q += 2) {
                            const uint2 t2 = __ldg(reinterpret_cast<const uint2 *>(ar + q));
                            av[q] = t2.x; av[q + 1] = t2.y;
                        }
                    } else {
#pragma unroll
                        for (int q = 0; q < KW; ++q) av[q] = __ldg(ar + q);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < KW; ++q) av[q] = 0u;
                }
#pragma unroll
                for (int g = 0; g < NIB; ++g)
                    naddr[g] = T_s + (uint32_t)(g * 16 + ((av[g >> 3] >> (4 * (g & 7))) & 15u)) * 4u;
            }
            // per 32-partner word w: transpose (BT), tabulate (T), look up.  Double buffered
            // (DB), one word's lookups overlap the next word's transposition (two barriers per
            // word); single buffered (when the second buffer would cost a CTA per SM), three
            for (int w = 0; w < W; ++w) {
                const int bw = DB ? (w & 1) : 0;
                uint32_t *BTw = BT + bw * 32 * KW;
                uint32_t *Tw = T + bw * NIB * 16;
                // transposed partner bits: warp j takes bit positions [j*PER, (j+1)*PER), all in
                // one 32-bit word of the partner vectors; lane pp keeps ballot pp
                {
                    const int t = 32 * w + lane;
                    constexpr int PER = 4 * KW;  // bits per warp (32*KW / 8 warps)
                    const int p0 = warp * PER;
                    // (PER = 24 at KW = 6: a warp's bits may span two words)
                    const uint32_t wlo = t < m ? sB[t * SBS + (p0 >> 5)] : 0u;
                    const uint32_t whi = (32 % PER == 0) ? wlo : t < m ? sB[t * SBS + ((p0 + PER - 1) >> 5)] : 0u;
                    uint32_t mine = 0u;
#pragma unroll
                    for (int pp = 0; pp < PER; ++pp) {
                        const int p = p0 + pp;
                        const uint32_t word = ((p >> 5) == (p0 >> 5)) ? wlo : whi;
                        const uint32_t bal = __ballot_sync(0xffffffffu, (word >> (p & 31)) & 1u);
                        if (lane == pp) mine = bal;
                    }
                    if (lane < PER) BTw[p0 + lane] = mine;
                }
                __syncthreads();
                for (int x = tid; x < NIB * 16; x += OWN_THREADS) {
                    const int g = x >> 4, v = x & 15;
                    uint32_t e = 0u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if ((v >> q) & 1) e ^= BTw[4 * g + q];
                    Tw[x] = e;
                }
                __syncthreads();
                if (k < m) {
                    const uint32_t toff = (uint32_t)(bw * NIB * 16 * 4);
                    uint32_t acc = 0u;
#pragma unroll
                    for (int g = 0; g < NIB; ++g) {
                        uint32_t e;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(naddr[g] + toff));
                        acc ^= e;
                    }
                    const int tend = min(32, m - 32 * w);
                    uint32_t bits = ~acc & (tend == 32 ? 0xffffffffu : ((1u << tend) - 1u));
                    if (k >> 5 == w) bits &= ~(1u << (k & 31));  // no self pair
                    out[(int64_t)k * W + w] = bits;
                }
                if (!DB) __syncthreads();
            }
            if (DB) __syncthreads();  // (the next row block reuses the buffers from word 0)
        }
        // ---- ownership: (c', k) for every color c' < c of every member's list.  Rectangular
        // lists: one thread per (member, slot) item, consecutive threads on consecutive slots
        // of a member (coalesced loads); ragged lists: warp per member.
        auto insert = [&](uint32_t cp, int k) {
            const uint32_t key = (cp << 12) | (uint32_t)k;
            uint32_t slot = mix32(cp) & (HS - 1);
            for (int probe = 0;; ++probe) {
                if (probe == HS) {
                    overflow = 1;
                    return;
                }
                const uint32_t prev = atomicCAS(&table[slot], 0u, key);
                if (prev == 0u) return;
                if ((prev >> 12) == cp) {
                    const int q = atomicAdd(&ncoll, 1);
                    if (q < OWN_COLL) coll[q] = (slot << 12) | (uint32_t)k;
                    else overflow = 1;
                    return;
                }
                slot = (slot + 1) & (HS - 1);
            }
        };
        if (o.direct) {
            // Leveled direct-mapped ownership: at level 1 every (c' < c, member k) writes k
            // into slot c' (last writer wins); after a barrier every writer whose k was
            // overwritten is a loser: it shares c' with the slot's winner (pair not owned by c)
            // and retries at the next level with the other losers.  Level by level each group
            // of members sharing c' yields every pair exactly once.  A slot is only read in
            // the round that just wrote it, and a member's colors are distinct, so the member
            // index alone identifies the surviving write (16-bit tags, no reset between colors).
            auto clear_pair = [&](int k1, int k2) {
                atomicAnd(&out[(int64_t)k1 * W + (k2 >> 5)], ~(1u << (k2 & 31)));
                atomicAnd(&out[(int64_t)k2 * W + (k1 >> 5)], ~(1u << (k1 & 31)));
            };
            const uint32_t items = (uint32_t)m * (uint32_t)o.L;
            if (tid == 0) nlose = 0;
            for (uint32_t e = tid; e < items; e += OWN_THREADS) {
                const int k = (int)__umulhi(e, o.l_magic);
                const int32_t cx = o.l16 ? (int32_t)sL16[e] : sL32[e];
                if (cx < c) dtab[cx] = (unsigned short)k;
            }
            __syncthreads();
            for (uint32_t e = tid; e < items; e += OWN_THREADS) {
                const int k = (int)__umulhi(e, o.l_magic);
                const int32_t cx = o.l16 ? (int32_t)sL16[e] : sL32[e];
                if (cx < c) {
                    const int w = dtab[cx];
                    if (w != k) {
                        clear_pair(k, w);
                        const int q = atomicAdd(&nlose, 1);
                        if (q < lcap) lA[q] = ((uint32_t)cx << 12) | (uint32_t)k;
                        else overflow = 2;
                    }
                }
            }
            __syncthreads();
            int nl = min(nlose, lcap);
            uint32_t *src = lA, *dst = lB;
            for (uint32_t level = 2; nl > 0; ++level) {
                if (level >= 64) {  // a color shared by 64+ members of one bucket: dedupe path
                    if (tid == 0) overflow = 3;
                    break;
                }
                __syncthreads();
                if (tid == 0) nlose = 0;
                for (int q = tid; q < nl; q += OWN_THREADS)
                    dtab[src[q] >> 12] = (unsigned short)(src[q] & 0xfffu);
                __syncthreads();
                for (int q = tid; q < nl; q += OWN_THREADS) {
                    const int w = dtab[src[q] >> 12];
                    const int k = (int)(src[q] & 0xfffu);
                    if (w != k) {
                        clear_pair(k, w);
                        dst[atomicAdd(&nlose, 1)] = src[q];
                    }
                }
                __syncthreads();
                nl = nlose;
                uint32_t *t = src;
                src = dst;
                dst = t;
            }
        } else if (o.bitmap) {
            // pass 1: every (member k, color c' < c) item sets bit c' of bm; an item that finds
            // the bit set marks c' in the filter.  Pass 2: the items whose color passes the
            // filter are listed; every pair of holders of one color is cleared below.
            constexpr int OWN_BATCH = 8;
            const uint32_t items = (uint32_t)m * (uint32_t)o.L;
            for (int pass = 0; pass < 2; ++pass) {
                for (uint32_t e0 = tid; e0 < items; e0 += OWN_BATCH * OWN_THREADS) {
                    int32_t cx[OWN_BATCH];
                    int kk[OWN_BATCH];
#pragma unroll
                    for (int u = 0; u < OWN_BATCH; ++u) {
                        const uint32_t e = e0 + (uint32_t)(u * OWN_THREADS);
                        const int k = (int)__umulhi(e, o.l_magic);
                        kk[u] = k;
                        cx[u] = e >= items ? INT_MAX
                              : !stage_lists ? __ldg(o.lrel + (int64_t)sid[k] * o.L + (e - (uint32_t)k * (uint32_t)o.L))
                              : o.l16 ? (int32_t)sL16[e] : sL32[e];
                    }
#pragma unroll
                    for (int u = 0; u < OWN_BATCH; ++u) {
                        if (cx[u] >= c) continue;
                        const uint32_t h = ((uint32_t)cx[u] * 0x9E3779B1u) >> 18;  // 14 bits
                        if (pass == 0) {
                            const uint32_t bit = 1u << (cx[u] & 31);
                            if (atomicOr(&bm[cx[u] >> 5], bit) & bit) atomicOr(&filt[h >> 5], 1u << (h & 31));
                        } else if ((filt[h >> 5] >> (h & 31)) & 1u) {
                            const int q = atomicAdd(&ncoll, 1);
                            if (q < OWN_BM_COLL) coll[q] = ((uint32_t)cx[u] << 12) | (uint32_t)kk[u];
                            else overflow = 1;
                        }
                    }
                }
                __syncthreads();
            }
        } else if (!o.loff) {
            // the list loads of OWN_BATCH items are issued together (the inserts' atomics
            // would otherwise serialise each load behind the previous item's insert)
            constexpr int OWN_BATCH = 8;
            const uint32_t items = (uint32_t)m * (uint32_t)o.L;
            for (uint32_t e0 = tid; e0 < items; e0 += OWN_BATCH * OWN_THREADS) {
                int32_t cx[OWN_BATCH];
                int kk[OWN_BATCH];
#pragma unroll
                for (int u = 0; u < OWN_BATCH; ++u) {
                    const uint32_t e = e0 + (uint32_t)(u * OWN_THREADS);
                    const int k = (int)__umulhi(e, o.l_magic);  // e / L (exact for e < 2^20)
                    kk[u] = k;
                    cx[u] = e >= items ? INT_MAX
                          : !stage_lists ? __ldg(o.lrel + (int64_t)sid[k] * o.L + (e - (uint32_t)k * (uint32_t)o.L))
                          : o.l16 ? (int32_t)sL16[e] : sL32[e];
                }
#pragma unroll
                for (int u = 0; u < OWN_BATCH; ++u)
                    if (cx[u] < c) insert((uint32_t)cx[u] + 1u, kk[u]);
            }
        } else {
            for (int k = warp; k < m; k += NWARPS) {
                const int32_t r = sid[k];
                for (int64_t x = o.loff[r] + lane; x < o.loff[r + 1]; x += 32) {
                    const int32_t cx = o.lrel[x];
                    if (cx < c) insert((uint32_t)cx + 1u, k);
                }
            }
        }
        __syncthreads();
        const int nc = o.direct ? 0 : min(ncoll, coll_cap);
        if (overflow && tid == 0) atomicMax(o.overflow, overflow);
        // every collision entry (a later holder k2 of a color c' < c) pairs with the first
        // holder (the table slot) and with the earlier collision entries of the same slot, so
        // each pair of a group sharing c' is cleared exactly once (groups are almost always
        // pairs: ~(L-1)^2/P of a bucket's pairs share a second color)
        if (o.bitmap) {  // every pair of holders of one color, once
            for (int q = tid; q < nc; q += OWN_THREADS) {
                const uint32_t cq = coll[q];
                const int k2 = (int)(cq & 0xfffu);
                for (int p = 0; p < q; ++p) {
                    const uint32_t cp = coll[p];
                    if ((cp >> 12) == (cq >> 12)) {
                        const int k0 = (int)(cp & 0xfffu);
                        atomicAnd(&out[(int64_t)k0 * W + (k2 >> 5)], ~(1u << (k2 & 31)));
                        atomicAnd(&out[(int64_t)k2 * W + (k0 >> 5)], ~(1u << (k0 & 31)));
                    }
                }
            }
        }
        for (int q = tid; q < (o.bitmap ? 0 : nc); q += OWN_THREADS) {
            const uint32_t cq = coll[q];
            const uint32_t slot = cq >> 12;
            const int k2 = (int)(cq & 0xfffu);
            const int k1 = (int)(table[slot] & 0xfffu);
            if (k1 != k2) {
                atomicAnd(&out[(int64_t)k1 * W + (k2 >> 5)], ~(1u << (k2 & 31)));
                atomicAnd(&out[(int64_t)k2 * W + (k1 >> 5)], ~(1u << (k1 & 31)));
            }
            for (int p = 0; p < q; ++p) {
                const uint32_t cp = coll[p];
                const int k0 = (int)(cp & 0xfffu);
                if ((cp >> 12) == slot && k0 != k2) {
                    atomicAnd(&out[(int64_t)k0 * W + (k2 >> 5)], ~(1u << (k2 & 31)));
                    atomicAnd(&out[(int64_t)k2 * W + (k0 >> 5)], ~(1u << (k0 & 31)));
                }
            }
        }
        __syncthreads();
        // the rows' degrees (K2c's popcounts, fused: the prep zeroed deg/degu): each mask row
        // is final once the ownership clears above are done; re-read at L2 (.cg), where the
        // clears' atomics landed
        if (o.deg) {
            for (int k = k_lo + tid; k < k_hi; k += OWN_THREADS) {
                const uint32_t *row = out + (int64_t)k * W;
                int cnt = 0, cntu = 0;
                for (int w = 0; w < W; ++w) {
                    const uint32_t x = __ldcg(row + w);
                    cnt += __popc(x);
                    const int d = k - 32 * w;  // partners t > k are the ids > the row's
                    const uint32_t up = d < 0 ? 0xffffffffu : (d >= 31 ? 0u : ~((2u << d) - 1u));
                    cntu += __popc(x & up);
                }
                if (cnt) atomicAdd(&o.deg[sid[k]], cnt);
                if (cntu) atomicAdd(&o.degu[sid[k]], cntu);
            }
        }
        // reset the hash table or the bitmaps (direct tags carry the color: nothing to reset)
        if (!o.direct) {
            for (int x = 4 * tid; x < state_words; x += 4 * OWN_THREADS)
                *reinterpret_cast<uint4 *>(table + x) = make_uint4(0u, 0u, 0u, 0u);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------
// K2c: degrees from owned masks (warp per row, lane per color slot)
// ---------------------------------------------------------------------------------------
__global__ void k_count_owned(RowArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = a.row_begin + gw; i < a.row_end; i += nw) {
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        int cnt = 0, cntu = 0;
        for (int s = lane; s < Li; s += 32) {
            const int c = a.lrel[lo + s];
            const int m = a.bstart[c + 1] - a.bstart[c];
            const int W = (m + 31) >> 5;
            const int k = a.posof[lo + s];
            const uint32_t *row = a.masks + a.maskoff[c] + (int64_t)k * W;
            for (int w = 0; w < W; ++w) {
                const uint32_t x = __ldg(row + w);
                cnt += __popc(x);
                const int d = k - 32 * w;  // partners t > k are the ids > i (bucket ascends)
                const uint32_t up = d < 0 ? 0xffffffffu : (d >= 31 ? 0u : ~((2u << d) - 1u));
                cntu += __popc(x & up);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            cnt += __shfl_down_sync(0xffffffffu, cnt, o);
            cntu += __shfl_down_sync(0xffffffffu, cntu, o);
        }
        if (lane == 0) {
            a.deg[i] = cnt;
            a.degu[i] = cntu;
        }
    }
}

size_t owned_smem(const OwnArgs &o, int kw) {
    return (size_t)(o.hash_slots + o.hash_slots / 2 + 2 * OWN_COLL + o.m_cap + (size_t)o.m_cap * kw) * 4;
}

template <int KW>
int run_owned(const BucketArgs &b, const OwnArgs &o, int sms, cudaStream_t s) {
    int per_sm = 0;
    const size_t smem = owned_smem(o, b.kw);
    allow_max_smem(k_owned_masks<KW>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_owned_masks<KW>, OWN_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms * 4, b.P));
    k_owned_masks<KW><<<(unsigned)grid, OWN_THREADS, smem, s>>>(b, o);
    return 1;
}

size_t owned_fr_smem(const OwnArgs &o, int kw, bool db = false) {
    const size_t state = o.direct ? (size_t)o.dtab_words + 2 * (size_t)(o.lcap > 0 ? o.lcap : OWN_LCAP)
                         : o.bitmap ? (size_t)owned_bitmap_words(o)
                                    : (size_t)o.hash_slots + OWN_COLL;
    const size_t lists = o.stage_lists ? (size_t)o.m_cap * o.L * (o.l16 ? 2 : 4) : 0;
    const size_t nb = db ? 2 : 1;
    return (state + ((o.m_cap + 3) & ~3) + nb * 8 * (size_t)kw * 16 + nb * 32 * (size_t)kw +
            (((size_t)o.m_cap * (kw >= 4 ? kw + 1 : kw) + 3) & ~(size_t)3)) * 4 +
           ((lists + 15) & ~(size_t)15);
}

// double-buffered tables unless the second buffer costs a CTA per SM
template <int KW>
int run_owned_fr(const BucketArgs &b, const OwnArgs &o, int sms, cudaStream_t s) {
    int per1 = 0, per2 = 0;
    const size_t smem1 = owned_fr_smem(o, KW, false), smem2 = owned_fr_smem(o, KW, true);
    allow_max_smem(k_owned_fr<KW, false>);
    allow_max_smem(k_owned_fr<KW, true>);
    prefer_max_shared(k_owned_fr<KW, false>);
    prefer_max_shared(k_owned_fr<KW, true>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per1, k_owned_fr<KW, false>, OWN_THREADS, smem1);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, k_owned_fr<KW, true>, OWN_THREADS, smem2);
    const bool db = per2 >= per1 && per2 >= 1;
    const int per_sm = std::max(1, db ? per2 : per1);
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms * 4, b.P));
    if (db) k_owned_fr<KW, true><<<(unsigned)grid, OWN_THREADS, smem2, s>>>(b, o);
    else k_owned_fr<KW, false><<<(unsigned)grid, OWN_THREADS, smem1, s>>>(b, o);
    return 1;
}

}  // namespace

// ownership state words of the bitmap mode (bitmap + filter + holders) and of the hash's
// collision list
int64_t owned_bitmap_words(const OwnArgs &o) { return (int64_t)o.bm_words + OWN_BM_FILTER + OWN_BM_COLL; }
int64_t owned_hash_coll() { return OWN_COLL; }

// dynamic shared memory the owned-mask kernel launch_owned_masks picks would request
size_t owned_masks_smem(const OwnArgs &o, int kw) {
    if (o.fr && (kw == 2 || kw == 4 || kw == 6 || kw == 8)) return owned_fr_smem(o, kw);
    return owned_smem(o, kw);
}

int launch_owned_masks(const BucketArgs &b, const OwnArgs &o, int sms, cudaStream_t s) {
    if (o.fr) {
        switch (b.kw) {
            case 2: return run_owned_fr<2>(b, o, sms, s);
            case 4: return run_owned_fr<4>(b, o, sms, s);
            case 6: return run_owned_fr<6>(b, o, sms, s);
            case 8: return run_owned_fr<8>(b, o, sms, s);
            default: break;
        }
    }
    switch (b.kw) {
        case 2: return run_owned<2>(b, o, sms, s);
        case 4: return run_owned<4>(b, o, sms, s);
        case 6: return run_owned<6>(b, o, sms, s);
        case 8: return run_owned<8>(b, o, sms, s);
        case 12: return run_owned<12>(b, o, sms, s);
        default: return run_owned<0>(b, o, sms, s);
    }
}

int launch_count_owned(const RowArgs &a, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    const int64_t warps = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((warps + 7) / 8, (int64_t)sms * 16));
    k_count_owned<<<(unsigned)grid, 256, 0, s>>>(a);
    return 1;
}

}  // namespace pcg
