// Owned bucket masks (K2a), popcount count pass (K2c) and merge fill pass (K2m).
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
constexpr int MERGE_WARPS = 4;

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
        if (b.runlen) {  // owned partners per member: the run lengths of the fill pass
            for (int k = tid; k < m; k += OWN_THREADS) {
                int cnt = 0;
                for (int w = 0; w < W; ++w) cnt += __popc(out[(int64_t)k * W + w]);
                b.runlen[b.bstart[c] + k] = cnt;
            }
        }
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
template <int KW>
__global__ void __launch_bounds__(OWN_THREADS) k_owned_fr(BucketArgs b, OwnArgs o) {
    constexpr int NIB = 8 * KW;
    extern __shared__ __align__(16) uint32_t osm[];
    const int HS = o.hash_slots;
    // ownership state: hash (large palettes) or a direct-mapped table over the colors
    uint32_t *table = osm;                                        // HS: (c'+1)<<12 | first k
    unsigned short *head = reinterpret_cast<unsigned short *>(osm + HS);  // HS: last coll + 1
    uint32_t *coll = osm + HS + HS / 2;                           // OWN_COLL: slot<<12 | k
    int32_t *link = reinterpret_cast<int32_t *>(coll + OWN_COLL); // OWN_COLL: previous in slot
    unsigned short *dtab = reinterpret_cast<unsigned short *>(osm);  // direct: P member tags
    uint32_t *lA = osm + o.dtab_words;                            // direct: losers (c'<<12|k)
    const int lcap = o.lcap > 0 ? o.lcap : OWN_LCAP;
    uint32_t *lB = lA + lcap;
    int32_t *sid = reinterpret_cast<int32_t *>(osm + (o.direct ? o.dtab_words + 2 * lcap
                                                               : HS + HS / 2 + 2 * OWN_COLL));
    uint32_t *T = reinterpret_cast<uint32_t *>(sid + ((o.m_cap + 3) & ~3));  // NIB*16 table
    uint32_t *BT = T + NIB * 16;                                  // 32*KW transposed bits
    uint32_t *sB = BT + 32 * KW;                                  // members' partner vectors
    // members' color lists (rectangular lists): u16 when the palette allows, else u32
    void *sLv = sB + o.m_cap * KW;
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
        for (int x = tid; x < HS + HS / 2; x += OWN_THREADS) osm[x] = 0u;
    }
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
            sB[x] = __ldg(b.B + (int64_t)sid[x / KW] * KW + x % KW);
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
#pragma unroll
                for (int q = 0; q < KW; ++q) av[q] = k < m ? __ldg(b.A + (int64_t)sid[k] * KW + q) : 0u;
#pragma unroll
                for (int g = 0; g < NIB; ++g)
                    naddr[g] = T_s + (uint32_t)(g * 16 + ((av[g >> 3] >> (4 * (g & 7))) & 15u)) * 4u;
            }
            for (int w = 0; w < W; ++w) {
                // transposed partner bits: warp j takes bit positions [j*4*KW, (j+1)*4*KW)
                {
                    const int t = 32 * w + lane;
                    constexpr int PER = 4 * KW;  // bits per warp (32*KW / 8 warps)
#pragma unroll
                    for (int pp = 0; pp < PER; ++pp) {
                        const int p = warp * PER + pp;
                        const uint32_t word = t < m ? sB[t * KW + (p >> 5)] : 0u;
                        const uint32_t bal = __ballot_sync(0xffffffffu, (word >> (p & 31)) & 1u);
                        if (lane == 0) BT[p] = bal;
                    }
                }
                __syncthreads();
                for (int x = tid; x < NIB * 16; x += OWN_THREADS) {
                    const int g = x >> 4, v = x & 15;
                    uint32_t e = 0u;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if ((v >> q) & 1) e ^= BT[4 * g + q];
                    T[x] = e;
                }
                __syncthreads();
                if (k < m) {
                    uint32_t acc = 0u;
#pragma unroll
                    for (int g = 0; g < NIB; ++g) {
                        uint32_t e;
                        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(e) : "r"(naddr[g]));
                        acc ^= e;
                    }
                    const int tend = min(32, m - 32 * w);
                    uint32_t bits = ~acc & (tend == 32 ? 0xffffffffu : ((1u << tend) - 1u));
                    if (k >> 5 == w) bits &= ~(1u << (k & 31));  // no self pair
                    out[(int64_t)k * W + w] = bits;
                }
                __syncthreads();
            }
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
                    if (q < OWN_COLL) {
                        coll[q] = (slot << 12) | (uint32_t)k;
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
        } else if (!o.loff) {
            const uint32_t items = (uint32_t)m * (uint32_t)o.L;
            for (uint32_t e = tid; e < items; e += OWN_THREADS) {
                const int k = (int)__umulhi(e, o.l_magic);  // e / L (exact for e < 2^20)
                const int32_t cx = !stage_lists ? o.lrel[(int64_t)sid[k] * o.L + (e - (uint32_t)k * (uint32_t)o.L)]
                                 : o.l16 ? (int32_t)sL16[e] : sL32[e];
                if (cx < c) insert((uint32_t)cx + 1u, k);
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
        const int nc = o.direct ? 0 : min(ncoll, OWN_COLL);
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
        if (b.runlen) {  // owned partners per member: the run lengths of the runs fill
            for (int k = tid; k < m; k += OWN_THREADS) {
                int cnt = 0;
                for (int w = 0; w < W; ++w) cnt += __popc(out[(int64_t)k * W + w]);
                b.runlen[b.bstart[c] + k] = cnt;
            }
        }
        // reset the hash table and the chain heads this color touched (direct tags carry the
        // color: nothing to reset)
        if (!o.direct) {
            for (int x = 4 * tid; x < HS; x += 4 * OWN_THREADS)
                *reinterpret_cast<uint4 *>(table + x) = make_uint4(0u, 0u, 0u, 0u);
            for (int q = tid; q < nc; q += OWN_THREADS) head[coll[q] >> 12] = 0;  // (16-bit store)
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

// ---------------------------------------------------------------------------------------
// K2m: fill by merging the row's disjoint runs (warp per row, shared memory merge path)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ int merge_split(const int32_t *A, int la, const int32_t *B, int lb,
                                           int d) {
    int lo = max(0, d - lb), hi = min(d, la);
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] < B[d - 1 - mid]) lo = mid + 1; else hi = mid;
    }
    return lo;
}

template <typename OutT>
__global__ void __launch_bounds__(MERGE_WARPS * 32) k_fill_merge(RowArgs a, MergeArgs g) {
    extern __shared__ __align__(16) int32_t msm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int cap = g.cap;
    int32_t *buf0 = msm + (size_t)warp * (2 * cap + 68);
    int32_t *buf1 = buf0 + cap;
    int32_t *roff = buf1 + cap;  // up to 33 run offsets (+ padding)
    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int64_t gw = blockIdx.x * (int64_t)MERGE_WARPS + warp;
    const int64_t nw = (int64_t)gridDim.x * MERGE_WARPS;
    for (int64_t i = a.row_begin + gw; i < a.row_end; i += nw) {
        const int deg = a.deg[i];
        if (deg == 0) continue;
        if (deg > cap) {  // too long for shared memory: the bitmap fill handles it
            if (lane == 0) g.heavy[atomicAdd(g.nheavy, 1)] = (int32_t)i;
            continue;
        }
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        // ---- decode: runs of the row's colors, ascending member ids where the owned bit is set
        int fillv = 0;
        for (int s = 0; s < Li; ++s) {
            if (lane == 0) roff[s] = fillv;
            const int c = a.lrel[lo + s];
            const int m = a.bstart[c + 1] - a.bstart[c];
            const int W = (m + 31) >> 5;
            const uint32_t *row = a.masks + a.maskoff[c] + (int64_t)a.posof[lo + s] * W;
            const int32_t *mem = a.bmemp + a.bpos[c];
            for (int w0 = 0; w0 < W; w0 += 8) {
                int32_t v[8];
                uint32_t mw[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const int w = w0 + u;
                    mw[u] = w < W ? __ldg(row + w) : 0u;
                    v[u] = (w < W && 32 * w + lane < m) ? __ldg(mem + 32 * w + lane) : 0;
                }
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const bool adm = (mw[u] >> lane) & 1u;
                    const uint32_t bal = __ballot_sync(0xffffffffu, adm);
                    if (adm) buf0[fillv + __popc(bal & ((1u << lane) - 1u))] = v[u];
                    fillv += __popc(bal);
                }
            }
        }
        if (lane == 0) roff[Li] = fillv;
        __syncwarp();
        // ---- merge tree: pairs of runs per level, merge path per lane
        int R = Li;
        int32_t *src = buf0, *dst = buf1;
        while (R > 1) {
            const int total = roff[R];
            const int olo = (int)((int64_t)total * lane / 32);
            const int ohi = (int)((int64_t)total * (lane + 1) / 32);
            // each lane finds the pair(s) its output range falls in and merges on its own,
            // so all lanes run their (equal-length) merge loops at the same time
            int o = olo;
            while (o < ohi) {
                int p = 0;  // last pair whose output starts at or before o
                for (int q = 1; 2 * q < R; ++q)
                    if (roff[2 * q] <= o) p = q;
                const int a0 = roff[2 * p], a1 = roff[min(2 * p + 1, R)];
                const int e = roff[min(2 * p + 2, R)];
                const int s1 = min(ohi, e);
                const int32_t *A = src + a0, *B = src + a1;
                const int la = a1 - a0, lb = e - a1;
                int ia = merge_split(A, la, B, lb, o - a0);
                int ib = (o - a0) - ia;
                int32_t xa = ia < la ? A[ia] : INT_MAX;
                int32_t xb = ib < lb ? B[ib] : INT_MAX;
                for (; o < s1; ++o) {
                    if (xa < xb) {
                        dst[o] = xa;
                        ++ia;
                        xa = ia < la ? A[ia] : INT_MAX;
                    } else {
                        dst[o] = xb;
                        ++ib;
                        xb = ib < lb ? B[ib] : INT_MAX;
                    }
                }
            }
            __syncwarp();
            const int R2 = (R + 1) >> 1;
            int nr = 0;
            if (lane <= R2) nr = roff[min(2 * lane, R)];
            __syncwarp();
            if (lane <= R2) roff[lane] = nr;
            __syncwarp();
            R = R2;
            int32_t *t = src;
            src = dst;
            dst = t;
        }
        // ---- coalesced store (compact ids when some rows have no conflicts)
        const int64_t base = a.rowoff[i] - a.out_base;
        for (int k = lane; k < deg; k += 32) {
            const int32_t j = src[k];
            out[base + k] = (OutT)(a.compact ? a.compact[j] : j);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------------------
// K2f: cooperative bitmap fill with owned masks (warp per row).  The warp walks one color
// bucket at a time: 32 consecutive members per coalesced load (a whole bucket slice per
// batch, all loads in flight), admitted members (owned-mask bit) compacted with a ballot, so
// the ids in lanes 0..k-1 ascend.  Equal bitmap words can then only sit in neighbouring
// lanes: two shuffles find them; unique words get a plain read-or-write, shared ones an
// atomic.  Rows come out of the interleaved harvest in ascending order.
// ---------------------------------------------------------------------------------------
constexpr int COOP_WARPS = 8;
constexpr int COOP_BATCH = 8;   // 32-member chunks per load batch
constexpr int COOP_STAGE = 1024;
constexpr int UNR_F = 8;    // run elements per lane per round (runs fill)

__device__ __forceinline__ uint32_t c_lds(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
__device__ __forceinline__ void c_sts(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ uint4 c_lds4(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr)
                 : "memory");
    return v;
}
__device__ __forceinline__ void c_sts4(uint32_t addr, uint4 v) {
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ int c_scan(int v, int lane, int &total) {
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    return x - v;
}

template <typename OutT>
__global__ void __launch_bounds__(COOP_WARPS * 32) k_fill_coop(RowArgs a) {
    extern __shared__ __align__(16) uint32_t csm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int WW = a.window >> 5;
    uint32_t *bm = csm + (size_t)warp * (WW + COOP_STAGE + 4 * a.slot_cap);
    int32_t *stage = reinterpret_cast<int32_t *>(bm + WW);
    int32_t *st = stage + COOP_STAGE;       // cursor
    int32_t *sm = st + a.slot_cap;          // bucket size
    int32_t *sb = sm + a.slot_cap;          // bucket base in bmemp
    int32_t *sw = sb + a.slot_cap;          // mask row offset (words) relative to masks
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(bm);
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    __syncwarp();
    OutT *out = reinterpret_cast<OutT *>(a.out);
    const uint32_t lt = (1u << lane) - 1u;
    const int64_t stride = (int64_t)gridDim.x * COOP_WARPS;
    for (int64_t ri = a.row_begin + (int64_t)blockIdx.x * COOP_WARPS + warp; ri < a.row_end;
         ri += stride) {
        const int64_t i = a.rows_list ? (int64_t)a.rows_list[ri] : ri;
        if (a.deg[i] == 0) continue;
        const int64_t lo = a.loff ? a.loff[i] : i * a.L;
        const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
        for (int s = lane; s < Li; s += 32) {
            const int c = a.lrel[lo + s];
            const int m = a.bstart[c + 1] - a.bstart[c];
            st[s] = 0;
            sm[s] = m;
            sb[s] = a.bpos[c];
            sw[s] = (int32_t)(a.maskoff[c] + (int64_t)a.posof[lo + s] * ((m + 31) >> 5));
        }
        __syncwarp();
        int64_t outpos = a.rowoff[i] - a.out_base;
        for (int32_t w0 = 0; w0 < a.n; w0 += a.window) {
            const int32_t w1 = (int32_t)min((int64_t)a.n, (int64_t)w0 + a.window);
            for (int s = 0; s < Li; ++s) {
                int t = st[s];
                const int m = sm[s];
                if (t >= m) continue;
                const int32_t *mem = a.bmemp + sb[s];
                const uint32_t *mrow = a.masks + sw[s];
                bool more = true;
                while (more) {
                    int32_t v[COOP_BATCH];
                    uint32_t mw[COOP_BATCH];
#pragma unroll
                    for (int u = 0; u < COOP_BATCH; ++u) {
                        const int p = t + 32 * u + lane;
                        const bool ok = p < m;
                        v[u] = ok ? __ldg(mem + p) : INT_MAX;
                        mw[u] = ok ? __ldg(mrow + (p >> 5)) : 0u;
                    }
#pragma unroll
                    for (int u = 0; u < COOP_BATCH; ++u) {
                        if (!more) break;
                        const int p = t + lane;
                        const bool in = v[u] < w1;
                        const int k = __popc(__ballot_sync(0xffffffffu, in));
                        const bool adm = in && ((mw[u] >> (p & 31)) & 1u);
                        const uint32_t am = __ballot_sync(0xffffffffu, adm);
                        const int na = __popc(am);
                        // lane l < na takes the l-th admitted id (ascending)
                        const int src = lane < na ? __fns(am, 0, lane + 1) : 0;
                        const int32_t id = __shfl_sync(0xffffffffu, v[u], src);
                        const bool act = lane < na;
                        const uint32_t off = (uint32_t)(id - w0);
                        const int32_t word = act ? (int32_t)(off >> 5) : -1 - lane;
                        const int32_t up = __shfl_up_sync(0xffffffffu, word, 1);
                        const int32_t dn = __shfl_down_sync(0xffffffffu, word, 1);
                        const bool dup = act && ((lane > 0 && up == word) || (lane < 31 && dn == word));
                        const uint32_t addr = bm_s + ((off >> 5) << 2);
                        const uint32_t bit = 1u << (off & 31);
                        if (act && !dup) c_sts(addr, c_lds(addr) | bit);
                        if (__any_sync(0xffffffffu, dup)) {
                            if (dup)
                                atomicOr(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(addr)), bit);
                        }
                        t += k;
                        more = (k == 32) && t < m;
                    }
                }
                if (lane == 0) st[s] = t;
                __syncwarp();
            }
            // ---- harvest: interleaved 16-byte chunks, ids staged then stored coalesced
            const int rows = WW >> 7;
            int fillv = 0;
            for (int it = 0; it < rows; ++it) {
                const int c = it * 32 + lane;
                const uint32_t addr = bm_s + (uint32_t)c * 16u;
                const uint4 q4 = c_lds4(addr);
                const int nb = __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
                int total;
                const int base = c_scan(nb, lane, total);
                if (total == 0) continue;
                const bool direct = total > COOP_STAGE;
                if (fillv > 0 && (direct || fillv + total > COOP_STAGE)) {
                    __syncwarp();
                    for (int k = lane; k < fillv; k += 32) out[outpos + k] = (OutT)stage[k];
                    outpos += fillv;
                    fillv = 0;
                    __syncwarp();
                }
                if (nb) {
                    c_sts4(addr, make_uint4(0u, 0u, 0u, 0u));
                    int64_t pos = direct ? outpos + base : fillv + base;
                    const uint32_t wv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        uint32_t wd = wv[u];
                        const int32_t jb = w0 + c * 128 + 32 * u;
                        while (wd) {
                            const int bb = __ffs(wd) - 1;
                            wd &= wd - 1u;
                            const int32_t j = jb + bb;
                            const int32_t val = a.compact ? a.compact[j] : j;
                            if (direct) out[pos++] = (OutT)val;
                            else stage[pos++] = val;
                        }
                    }
                }
                if (direct) outpos += total;
                else fillv += total;
            }
            __syncwarp();
            for (int k = lane; k < fillv; k += 32) out[outpos + k] = (OutT)stage[k];
            outpos += fillv;
            __syncwarp();
        }
    }
}

template <typename OutT>
int run_coop(const RowArgs &a, int sms, cudaStream_t s) {
    const size_t per_warp = (size_t)((a.window >> 5) + COOP_STAGE + 4 * a.slot_cap) * 4;
    const size_t smem = per_warp * COOP_WARPS;
    allow_max_smem(k_fill_coop<OutT>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fill_coop<OutT>, COOP_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)per_sm * sms, (rows + COOP_WARPS - 1) / COOP_WARPS));
    k_fill_coop<OutT><<<(unsigned)grid, COOP_WARPS * 32, smem, s>>>(a);
    return 1;
}


// ---------------------------------------------------------------------------------------
// Owned partner runs: for every bucket entry (color c, member k) the ascending ids of its
// owned admitted partners, at a 16-byte aligned offset (TMA bulk copies need it).  Warp per
// color; 32 bucket positions per step, ballot-compacted, coalesced stores.
// ---------------------------------------------------------------------------------------
constexpr int RUN_WARPS = 8;

__global__ void __launch_bounds__(RUN_WARPS * 32) k_write_runs(BucketArgs b, RunArgs r) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)RUN_WARPS + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * RUN_WARPS;
    for (int64_t c = gw; c < b.P; c += nw) {
        const int m = b.bstart[c + 1] - b.bstart[c];
        if (m < 2) continue;
        const int W = (m + 31) >> 5;
        const int32_t *mem = b.bmemp + b.bpos[c];
        const uint32_t *mk = b.masks + b.maskoff[c];
        for (int k = 0; k < m; ++k) {
            const int64_t pos = b.bstart[c] + k;
            int32_t *dst = r.runs + r.runoff[pos];
            int cnt = 0;
            for (int w = 0; w < W; ++w) {
                const uint32_t word = __ldg(mk + (int64_t)k * W + w);  // broadcast
                if (word == 0u) continue;
                const int t = 32 * w + lane;
                const bool keep = (word >> lane) & 1u;
                const int32_t id = keep ? __ldg(mem + t) : 0;
                if (keep) dst[cnt + __popc(word & ((1u << lane) - 1u))] = id;
                cnt += __popc(word);
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// Fill from owned runs (warp per row).  Lanes s < L issue one TMA bulk copy each (their
// run) into the warp's shared staging buffer, completing on an mbarrier; the next row is
// staged into the other buffer while this one is sorted.  Lanes then walk their run in
// shared memory and mark partners in the window bitmap; the interleaved harvest emits the
// row in ascending order (runs are disjoint: no dedupe needed).
// ---------------------------------------------------------------------------------------
constexpr int FR_W = 4;  // warps per block

__device__ __forceinline__ void mbar_init(uint32_t mbar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "\t@!p bra W%=;\n\t}" ::"r"(mbar),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void tma_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(mbar)
        : "memory");
}

struct RowStage {
    int off, len;     // this lane's run inside the buffer (ids)
    int deg;          // row total (warp-uniform)
};

// Issue the TMA copies of row i into buffer `buf_s` (shared byte address).  Returns the
// lane's run geometry.  deg == -1 marks a row too long for the buffer.
__device__ __forceinline__ RowStage stage_row(const RowArgs &a, const RunArgs &r, int64_t i,
                                              uint32_t buf_s, uint32_t mbar, int lane) {
    RowStage g{0, 0, 0};
    const int64_t lo = a.loff ? a.loff[i] : i * a.L;
    const int Li = (int)((a.loff ? a.loff[i + 1] : lo + a.L) - lo);
    int64_t src = 0;
    int len = 0;
    if (lane < Li) {
        const int c = a.lrel[lo + lane];
        const int64_t pos = a.bstart[c] + a.posof[lo + lane];
        len = r.runlen[pos];
        src = r.runoff[pos];
    }
    const int padded = (len + 3) & ~3;
    int total;
    int x = padded;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    total = __shfl_sync(0xffffffffu, x, 31);
    const int off = x - padded;
    g.off = off;
    g.len = len;
    g.deg = total > r.cap ? -1 : total;
    if (g.deg > 0) {
        if (lane == 0) mbar_expect(mbar, (uint32_t)total * 4u);
        __syncwarp();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (padded > 0) tma_load(buf_s + (uint32_t)off * 4u, r.runs + src, (uint32_t)padded * 4u, mbar);
    }
    return g;
}

template <typename OutT>
__global__ void __launch_bounds__(FR_W * 32) k_fill_runs(RowArgs a, RunArgs r) {
    extern __shared__ __align__(16) uint32_t fsm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int WW = a.window >> 5;
    const size_t per_warp = (size_t)2 * r.cap + WW + 32 + COOP_STAGE + 4;
    uint32_t *base = fsm + (size_t)warp * per_warp;
    int32_t *buf0 = reinterpret_cast<int32_t *>(base);
    uint32_t *bm = base + 2 * r.cap;
    int32_t *stage = reinterpret_cast<int32_t *>(bm + WW + 32);
    uint64_t *mb = reinterpret_cast<uint64_t *>(stage + COOP_STAGE);
    const uint32_t bufs_s = (uint32_t)__cvta_generic_to_shared(buf0);
    const uint32_t bm_s = (uint32_t)__cvta_generic_to_shared(bm);
    const uint32_t dummy_s = bm_s + (uint32_t)(WW + lane) * 4u;
    const uint32_t mb_s = (uint32_t)__cvta_generic_to_shared(mb);
    for (int k = lane; k < WW; k += 32) bm[k] = 0u;
    if (lane == 0) {
        mbar_init(mb_s);
        mbar_init(mb_s + 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    OutT *out = reinterpret_cast<OutT *>(a.out);
    const int64_t stride = (int64_t)gridDim.x * FR_W;
    int64_t ri = a.row_begin + (int64_t)blockIdx.x * FR_W + warp;
    uint32_t phase[2] = {0u, 0u};
    int b = 0;
    RowStage cur{0, 0, 0};
    if (ri < a.row_end) cur = stage_row(a, r, ri, bufs_s, mb_s, lane);
    for (; ri < a.row_end; ri += stride) {
        const int64_t i = ri;
        // prefetch the next row into the other buffer
        RowStage nxt{0, 0, 0};
        const int64_t rn = ri + stride;
        if (rn < a.row_end)
            nxt = stage_row(a, r, rn, bufs_s + (uint32_t)((b ^ 1) * r.cap) * 4u, mb_s + 8 * (b ^ 1), lane);
        if (cur.deg < 0) {  // too long for the staging buffer: bitmap fallback pass
            if (lane == 0) r.heavy[atomicAdd(r.nheavy, 1)] = (int32_t)i;
        } else if (cur.deg > 0) {
            mbar_wait(mb_s + 8 * b, phase[b]);
            phase[b] ^= 1u;
            const int32_t *buf = buf0 + b * r.cap;
            int t = 0;
            int64_t outpos = a.rowoff[i] - a.out_base;
            for (int32_t w0 = 0; w0 < a.n; w0 += a.window) {
                const int32_t w1 = (int32_t)min((int64_t)a.n, (int64_t)w0 + a.window);
                bool go = t < cur.len;
                while (__any_sync(0xffffffffu, go)) {
                    uint32_t addr[UNR_F], bit[UNR_F];
                    int k = 0;
#pragma unroll
                    for (int u = 0; u < UNR_F; ++u) {
                        const int32_t v = (go && t + u < cur.len) ? buf[cur.off + t + u] : INT_MAX;
                        const bool in = v < w1;
                        k += in ? 1 : 0;
                        const uint32_t off = (uint32_t)(v - w0);
                        addr[u] = in ? bm_s + ((off >> 5) << 2) : dummy_s;
                        bit[u] = in ? (1u << (off & 31)) : 0u;
                    }
                    t += k;
                    go = go && k == UNR_F && t < cur.len;
                    // mark (plain RMW + verify; atomics only for lost bits)
                    uint32_t old[UNR_F];
#pragma unroll
                    for (int u = 0; u < UNR_F; ++u) old[u] = bit[u] ? c_lds(addr[u]) : 0u;
#pragma unroll
                    for (int u = 0; u < UNR_F; ++u)
                        if (bit[u]) c_sts(addr[u], old[u] | bit[u]);
                    __syncwarp();
                    uint32_t lost = 0u;
#pragma unroll
                    for (int u = 0; u < UNR_F; ++u) {
                        old[u] = bit[u] ? (bit[u] & ~c_lds(addr[u])) : 0u;
                        lost |= old[u];
                    }
                    if (__any_sync(0xffffffffu, lost != 0u)) {
#pragma unroll
                        for (int u = 0; u < UNR_F; ++u)
                            if (old[u])
                                atomicOr(reinterpret_cast<uint32_t *>(__cvta_shared_to_generic(addr[u])), old[u]);
                    }
                    __syncwarp();
                }
                // harvest: interleaved chunks, staged, coalesced stores
                const int rows = WW >> 7;
                int fillv = 0;
                for (int it = 0; it < rows; ++it) {
                    const int cc = it * 32 + lane;
                    const uint32_t ad = bm_s + (uint32_t)cc * 16u;
                    const uint4 q4 = c_lds4(ad);
                    const int nb = __popc(q4.x) + __popc(q4.y) + __popc(q4.z) + __popc(q4.w);
                    int total;
                    const int bse = c_scan(nb, lane, total);
                    if (total == 0) continue;
                    const bool direct = total > COOP_STAGE;
                    if (fillv > 0 && (direct || fillv + total > COOP_STAGE)) {
                        __syncwarp();
                        for (int q = lane; q < fillv; q += 32) out[outpos + q] = (OutT)stage[q];
                        outpos += fillv;
                        fillv = 0;
                        __syncwarp();
                    }
                    if (nb) {
                        c_sts4(ad, make_uint4(0u, 0u, 0u, 0u));
                        int64_t pos = direct ? outpos + bse : fillv + bse;
                        const uint32_t wv[4] = {q4.x, q4.y, q4.z, q4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            uint32_t wd = wv[u];
                            const int32_t jb = w0 + cc * 128 + 32 * u;
                            while (wd) {
                                const int bb = __ffs(wd) - 1;
                                wd &= wd - 1u;
                                const int32_t j = jb + bb;
                                const int32_t val = a.compact ? a.compact[j] : j;
                                if (direct) out[pos++] = (OutT)val;
                                else stage[pos++] = val;
                            }
                        }
                    }
                    if (direct) outpos += total;
                    else fillv += total;
                }
                __syncwarp();
                for (int q = lane; q < fillv; q += 32) out[outpos + q] = (OutT)stage[q];
                outpos += fillv;
                __syncwarp();
                if (!__any_sync(0xffffffffu, t < cur.len)) break;  // row done before n
            }
        }
        __syncwarp();
        cur = nxt;
        b ^= 1;
    }
}

template <typename OutT>
int run_fill_runs(const RowArgs &a, const RunArgs &r, int sms, cudaStream_t s) {
    const size_t per_warp = ((size_t)2 * r.cap + (a.window >> 5) + 32 + COOP_STAGE + 4) * 4;
    const size_t smem = per_warp * FR_W;
    allow_max_smem(k_fill_runs<OutT>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fill_runs<OutT>, FR_W * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)per_sm * sms, (rows + FR_W - 1) / FR_W));
    k_fill_runs<OutT><<<(unsigned)grid, FR_W * 32, smem, s>>>(a, r);
    return 1;
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

size_t owned_fr_smem(const OwnArgs &o, int kw) {
    const size_t state = o.direct ? (size_t)o.dtab_words + 2 * (size_t)(o.lcap > 0 ? o.lcap : OWN_LCAP)
                                  : (size_t)o.hash_slots + o.hash_slots / 2 + 2 * OWN_COLL;
    const size_t lists = o.stage_lists ? (size_t)o.m_cap * o.L * (o.l16 ? 2 : 4) : 0;
    return (state + ((o.m_cap + 3) & ~3) + 8 * (size_t)kw * 16 + 32 * (size_t)kw + (size_t)o.m_cap * kw) * 4 +
           ((lists + 15) & ~(size_t)15);
}

template <int KW>
int run_owned_fr(const BucketArgs &b, const OwnArgs &o, int sms, cudaStream_t s) {
    int per_sm = 0;
    const size_t smem = owned_fr_smem(o, KW);
    allow_max_smem(k_owned_fr<KW>);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_owned_fr<KW>, OWN_THREADS, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms * 4, b.P));
    k_owned_fr<KW><<<(unsigned)grid, OWN_THREADS, smem, s>>>(b, o);
    return 1;
}

template <typename OutT>
int run_merge(const RowArgs &a, const MergeArgs &g, int sms, cudaStream_t s) {
    const size_t smem = (size_t)MERGE_WARPS * (2 * g.cap + 68) * 4;
    allow_max_smem(k_fill_merge<OutT>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fill_merge<OutT>, MERGE_WARPS * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t rows = a.row_end - a.row_begin;
    const int64_t grid = std::max<int64_t>(
        1, std::min<int64_t>((int64_t)per_sm * sms, (rows + MERGE_WARPS - 1) / MERGE_WARPS));
    k_fill_merge<OutT><<<(unsigned)grid, MERGE_WARPS * 32, smem, s>>>(a, g);
    return 1;
}

}  // namespace

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

int launch_fill_merge(const RowArgs &a, const MergeArgs &g, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    return out64 ? run_merge<int64_t>(a, g, sms, s) : run_merge<int32_t>(a, g, sms, s);
}

int merge_smem_bytes(int cap) { return MERGE_WARPS * (2 * cap + 68) * 4; }

int launch_write_runs(const BucketArgs &b, const RunArgs &r, int sms, cudaStream_t s) {
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((b.P + RUN_WARPS - 1) / RUN_WARPS,
                                                                (int64_t)sms * 8));
    k_write_runs<<<(unsigned)grid, RUN_WARPS * 32, 0, s>>>(b, r);
    return 1;
}

int launch_fill_runs(const RowArgs &a, const RunArgs &r, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    return out64 ? run_fill_runs<int64_t>(a, r, sms, s) : run_fill_runs<int32_t>(a, r, sms, s);
}

int launch_fill_coop(const RowArgs &a, bool out64, int sms, cudaStream_t s) {
    if (a.row_end <= a.row_begin) return 0;
    return out64 ? run_coop<int64_t>(a, sms, s) : run_coop<int32_t>(a, sms, s);
}

}  // namespace pcg
