// K1 with 8-bit slices (k_commute_fr8) — the commuting-pair count over the upper triangle
// (view_edges_scanned, conflict.py:78,115; predicate pauli.py:258-268 / graph.py:335-336),
// four Russians over GF(2) like k_commute_fr6, with one byte of the row per lookup.
//
// Bound: shared-memory bytes per pair.  A lookup returns one table entry of EB bytes = the
// XOR of the partner bit-rows selected by one 8-bit slice of the row, for 8*EB partners.
// With S = K/8 slices a pair costs S*EB/(8*EB) = K/64 bytes: 2.0 B at q = 64 (6-bit slices:
// 2.75 B), 4.0 B at q = 128 (4-bit slices: 8 B).
//
// Why this fits: a 256-entry table per slice is 4x the 6-bit one, so the entry shrinks to
// 32 bytes (256 partners, two lanes x LDS.128) at K <= 192 and to 16 bytes (128 partners,
// one lane) at K = 256: S x 256 x EB = 64/128/192/128 KB at K = 64/128/192/256.
//
// Why it stays conflict-free with data-dependent entries: an LDS.128 is served a quarter
// warp (8 lanes, 128 bytes) per wavefront.  Entry (s, e) sits at  e*S*EB + s*EB,  so its
// bank group (address mod 128) depends only on the slice s, never on the entry e.  The RPQ
// rows of a quarter warp (4 at EB = 32, 8 at EB = 16) look up DIFFERENT slices at each step:
// row g of the quarter takes slice (u + g) mod S at step u (its K-bit vector rotated right by
// 8g bits once per row), so the quarter's lanes cover the 128 bytes exactly once.
//
// Row work per lookup: one PRMT (the byte), one LEA (the address), one LDS.128, and the XOR
// into the 128-partner accumulator (LOP3, two entries at a time).  Table rebuilds happen once
// per partner block a CTA visits; the blocks are visited folded (0, njb-1, 1, njb-2, ...), so
// every CTA's share of the work items spans ~2*njb/grid blocks (~27 at 1M rows): negligible.
#include <algorithm>

#include "pcg_internal.cuh"

namespace pcg {

namespace {


__host__ __device__ constexpr int ctz_c(int k) { return (k & 1) ? 0 : 1 + ctz_c(k >> 1); }

template <int KW>
struct Fr8Geom {
    static constexpr int K = 32 * KW;
    static constexpr int S = K / 8;                   // slices (tables)
    static constexpr int EB = KW <= 6 ? 32 : 16;      // entry bytes
    static constexpr int JB = 8 * EB;                 // partners per block
    static constexpr int LPR = EB / 16;               // lanes per row
    static constexpr int RPQ = 8 / LPR;               // rows per quarter warp
    static constexpr int RPW = 32 / LPR;              // rows per warp
    static constexpr int STRIDE = S * EB;             // bytes per entry index e
    static constexpr int BTW = JB / 32;               // 32-partner words per bit row
    static constexpr int BTS = BTW + 1;               // padded bit-row stride (words)
    static constexpr size_t TBL = (size_t)256 * STRIDE;
    static constexpr size_t SMEM = TBL + (size_t)K * BTS * 4 + 128;
};

__device__ __forceinline__ void lds128(uint32_t addr, uint32_t &a, uint32_t &b, uint32_t &c,
                                       uint32_t &d) {
    asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "r"(addr));
}

template <int KW, int FR8_WARPS>
__global__ void __launch_bounds__(FR8_WARPS * 32, 1) k_commute_fr8(
    const uint32_t *__restrict__ A, const uint32_t *__restrict__ B, int64_t n,
    const int64_t *__restrict__ item_start, int64_t njb, int32_t ichunk, int64_t item0,
    int64_t item1, unsigned long long *__restrict__ anti) {
    using G = Fr8Geom<KW>;
    constexpr int S = G::S, EB = G::EB, JB = G::JB, LPR = G::LPR, RPQ = G::RPQ,
                  RPW = G::RPW, STRIDE = G::STRIDE, BTW = G::BTW, BTS = G::BTS;
    constexpr int NT = FR8_WARPS * 32;
    extern __shared__ __align__(128) uint32_t smem[];
    __shared__ unsigned long long red[FR8_WARPS];
    const uint32_t smem_s = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t tbl_s = (smem_s + 127u) & ~127u;  // 128-byte aligned: bank group = s
    char *tbl = reinterpret_cast<char *>(smem) + (tbl_s - smem_s);
    uint32_t *bt = reinterpret_cast<uint32_t *>(tbl + G::TBL);  // K bit rows x BTS words

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int rsub = lane / LPR;         // row of this lane within the warp's RPW rows
    const int g = rsub % RPQ;            // row within the quarter warp: slice rotation
    const int h = lane % LPR;            // 16-byte part of the entry (128 partners)
    // address of slice (u + g) mod S, entry 0, this lane's part; the last RPQ-1 steps wrap
    const uint32_t pre0 = tbl_s + (uint32_t)(g * EB + h * 16);
    uint32_t prew[RPQ - 1];
#pragma unroll
    for (int k = 0; k < RPQ - 1; ++k) {
        const int u = S - RPQ + 1 + k;
        prew[k] = pre0 + (uint32_t)(u * EB) - (g >= S - u ? (uint32_t)STRIDE : 0u);
    }

    const int64_t nitems = item1 - item0;
    const int64_t my0 = item0 + nitems * blockIdx.x / gridDim.x;
    const int64_t my1 = item0 + nitems * (blockIdx.x + 1) / gridDim.x;
    int64_t cur_jb = -1;
    unsigned long long local = 0;

    // visit index of the first item (binary search once), then advanced item by item
    int64_t vis = 0;
    {
        int64_t hi = njb;
        while (hi - vis > 1) {
            const int64_t mid = (vis + hi) >> 1;
            if (item_start[mid] <= my0) vis = mid; else hi = mid;
        }
    }
    for (int64_t it = my0; it < my1; ++it) {
        while (item_start[vis + 1] <= it) ++vis;
        const int64_t jb = fr8_fold(vis, njb), ic = it - item_start[vis];
        if (jb != cur_jb) {
            __syncthreads();  // previous tables no longer in use
            // phase A: partner bit rows  bt[k][w] bit t = bit k of B[jb*JB + 32w + t]
            for (int w = warp; w < BTW; w += FR8_WARPS) {
                const uint32_t *bj = B + (jb * JB + 32 * w + lane) * KW;
                uint32_t v[KW];
#pragma unroll
                for (int k = 0; k < KW; ++k) v[k] = __ldg(bj + k);
#pragma unroll
                for (int k = 0; k < KW; ++k) {
                    uint32_t mine = 0;
#pragma unroll
                    for (int sb = 0; sb < 32; ++sb) {
                        const uint32_t word = __ballot_sync(0xffffffffu, (v[k] >> sb) & 1u);
                        if (lane == sb) mine = word;
                    }
                    bt[(32 * k + lane) * BTS + w] = mine;
                }
            }
            __syncthreads();
            // phase B: entry (s, e) word w = XOR of bit rows 8s+b for the set bits b of e.
            // Thread = (w, s, part); a part covers 256/P entries in Gray-code order.
            {
                constexpr int UNITS = S * BTW;
                constexpr int P = NT / UNITS >= 8 ? 8 : NT / UNITS >= 4 ? 4 : NT / UNITS >= 2 ? 2 : 1;
                constexpr int EPP = 256 / P;  // entries per part
                constexpr int LB = EPP == 32 ? 5 : EPP == 64 ? 6 : EPP == 128 ? 7 : 8;
                for (int t = threadIdx.x; t < UNITS * P; t += NT) {
                    const int w = t % BTW, s = (t / BTW) % S, part = t / UNITS;
                    const uint32_t *rb = bt + 8 * s * BTS + w;  // bit row 8s+b at rb[b*BTS]
                    uint32_t val = 0;
#pragma unroll
                    for (int b = LB; b < 8; ++b) val ^= ((part >> (b - LB)) & 1) ? rb[b * BTS] : 0u;
                    char *dst = tbl + (size_t)part * EPP * STRIDE + s * EB + w * 4;
#pragma unroll 32
                    for (int k = 0; k < EPP; ++k) {
                        if (k) val ^= rb[ctz_c(k) * BTS];
                        const int e = k ^ (k >> 1);
                        *reinterpret_cast<uint32_t *>(dst + (size_t)e * STRIDE) = val;
                    }
                }
            }
            __syncthreads();
            cur_jb = jb;
        }
        const int64_t jlast = min(n, (jb + 1) * (int64_t)JB);  // exclusive
        const int64_t i0 = ic * ichunk;
        const int64_t i1 = min(i0 + ichunk, jlast);
        const int64_t jbase = jb * JB + 128 * h;
        // the row's bits for the next iteration are loaded one iteration ahead (an L2 round
        // trip per 16 lookups would otherwise be exposed)
        uint32_t an[KW];
        auto load_row = [&](int64_t i) {
            if (i < i1) {
                if constexpr (KW % 4 == 0) {  // 16-byte aligned rows: LDG.128
#pragma unroll
                    for (int k = 0; k < KW; k += 4) {
                        const uint4 av = __ldg(reinterpret_cast<const uint4 *>(A + i * KW + k));
                        an[k] = av.x;
                        an[k + 1] = av.y;
                        an[k + 2] = av.z;
                        an[k + 3] = av.w;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < KW; k += 2) {
                        const uint2 av = __ldg(reinterpret_cast<const uint2 *>(A + i * KW + k));
                        an[k] = av.x;
                        an[k + 1] = av.y;
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < KW; ++k) an[k] = 0u;
            }
        };
        load_row(i0 + RPW * warp + rsub);
        for (int64_t ib = i0 + RPW * warp; ib < i1; ib += RPW * FR8_WARPS) {
            const int64_t i = ib + rsub;
            const bool live = i < i1;
            uint32_t a[KW];
#pragma unroll
            for (int k = 0; k < KW; ++k) a[k] = an[k];
            load_row(i + RPW * FR8_WARPS);
            // rotate right by 8g bits (g < RPQ <= 8): whole word first when g >= 4
            uint32_t r[KW];
            if constexpr (RPQ > 4) {
                const bool wr = g >= 4;
#pragma unroll
                for (int k = 0; k < KW; ++k) r[k] = wr ? a[(k + 1) % KW] : a[k];
#pragma unroll
                for (int k = 0; k < KW; ++k) a[k] = r[k];
            }
            const uint32_t sh = 8u * (uint32_t)(g & 3);
#pragma unroll
            for (int k = 0; k < KW; ++k) r[k] = __funnelshift_r(a[k], a[(k + 1) % KW], sh);
            uint32_t acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
#pragma unroll
            for (int u = 0; u < S; u += 2) {
                uint32_t ad[2];
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    const int uu = u + v;
                    const uint32_t byte = __byte_perm(r[uu >> 2], 0u, 0x4440u | (uint32_t)(uu & 3));
                    const uint32_t base = uu <= S - RPQ ? pre0 + (uint32_t)(uu * EB)
                                                        : prew[uu - (S - RPQ + 1)];
                    ad[v] = base + byte * (uint32_t)STRIDE;
                }
                uint32_t e0, e1, e2, e3, f0, f1, f2, f3;
                lds128(ad[0], e0, e1, e2, e3);
                lds128(ad[1], f0, f1, f2, f3);
                acc0 ^= e0 ^ f0;
                acc1 ^= e1 ^ f1;
                acc2 ^= e2 ^ f2;
                acc3 ^= e3 ^ f3;
            }
            if (ib + RPW <= min(i1, jb * (int64_t)JB)) {
                // the warp's rows are all live and below the block: every partner counts
                local += (uint32_t)(__popc(acc0) + __popc(acc1) + __popc(acc2) + __popc(acc3));
            } else if (live) {
                // partners j = jbase + 32w + t with j > i
                const uint32_t accw[4] = {acc0, acc1, acc2, acc3};
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    const int64_t d = i - (jbase + 32 * w);
                    const uint32_t m = d < 0 ? 0xffffffffu : (d >= 31 ? 0u : ~((2u << d) - 1u));
                    local += __popc(accw[w] & m);
                }
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_down_sync(0xffffffffu, local, o);
    if (lane == 0) red[warp] = local;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < FR8_WARPS; ++w) s += red[w];
        if (s) atomicAdd(anti, s);
    }
}

template <int KW, int NW>
int run_fr8_w(const uint32_t *A, const uint32_t *B, int64_t n, const int64_t *item_start,
              int64_t njb, int32_t ichunk, int64_t item0, int64_t item1,
              unsigned long long *anti, int sms, cudaStream_t s) {
    const size_t smem = Fr8Geom<KW>::SMEM;
    allow_max_smem(k_commute_fr8<KW, NW>);
    prefer_max_shared(k_commute_fr8<KW, NW>);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_commute_fr8<KW, NW>, NW * 32, smem);
    if (per_sm < 1) per_sm = 1;
    const int64_t grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * sms, item1 - item0));
    k_commute_fr8<KW, NW><<<(unsigned)grid, NW * 32, smem, s>>>(A, B, n, item_start, njb, ichunk,
                                                               item0, item1, anti);
    return 1;
}

// 16 warps (the whole register file) when K1 runs alone; 8 when it shares the SMs with the
// row passes (k1_async): half the registers stay free for their CTAs
template <int KW>
int run_fr8(const uint32_t *A, const uint32_t *B, int64_t n, const int64_t *item_start,
            int64_t njb, int32_t ichunk, int64_t item0, int64_t item1,
            unsigned long long *anti, int sms, int warps, cudaStream_t s) {
    if (warps == 8)
        return run_fr8_w<KW, 8>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
    return run_fr8_w<KW, 16>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, s);
}

}  // namespace

bool fr8_supported(int32_t kw) { return kw == 2 || kw == 4 || kw == 6 || kw == 8; }

int fr8_jb(int32_t kw) {
    switch (kw) {
        case 2: return Fr8Geom<2>::JB;
        case 4: return Fr8Geom<4>::JB;
        case 6: return Fr8Geom<6>::JB;
        case 8: return Fr8Geom<8>::JB;
        default: return 0;
    }
}

int launch_commute_fr8_items(const uint32_t *A, const uint32_t *B, int32_t kw, int64_t n,
                             const int64_t *item_start, int64_t njb, int32_t ichunk,
                             int64_t item0, int64_t item1, unsigned long long *anti, int sms,
                             int warps, cudaStream_t s) {
    if (item1 <= item0) return 0;
    switch (kw) {
        case 2: return run_fr8<2>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, warps, s);
        case 4: return run_fr8<4>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, warps, s);
        case 6: return run_fr8<6>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, warps, s);
        case 8: return run_fr8<8>(A, B, n, item_start, njb, ichunk, item0, item1, anti, sms, warps, s);
        default: return 0;
    }
}

}  // namespace pcg
