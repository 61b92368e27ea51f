// fg_knn_tile.cuh -- binned_select_knn forward, lane-per-query tile path
// (replaces pyx:188-329 for the common case: every coordinate binned, d <= 4,
// no direction mask / max_radius2 / exhaustive, float32 distances).
//
// Why a second kernel: the warp-per-query search (fg_knn_impl.cuh) spends
// ~3.9k warp instructions per query on per-query bookkeeping (region
// enumeration, span flattening, warp-wide top-k) for ~300 candidates.  Here
// the bookkeeping is paid once per TILE of up to 32 spatially compact queries
// and every candidate is evaluated by all 32 lanes at once (one lane = one
// query), so a candidate costs ~10 warp instructions for 32 (query, candidate)
// pairs.
//
// * tiles (k_tiles).  Lead cells (all binned dims but the last) are grouped in
//   2^(DB-1) blocks; along the last dim a block's cell columns are cut greedily
//   into segments of <= 32 points.  A tile = one segment: at most 32 queries in
//   a box of about 2 x 2 x 2 x 3 cells (north_star), emitted to a tile list.
// * per tile (k_tile_search, one warp, tiles fetched dynamically):
//   - lane l takes the l-th point of the tile (sorted order), q, cell coords;
//   - radius hint: density of the 4^(DB-1)-row neighbourhood of the block gives
//     the expected need-th neighbour distance r_k; per lane r = alpha r_k f^(-1/d)
//     where f = prod over dims of (1 - cap_lo - cap_hi) is the fraction of the
//     ball inside the split's grid box (cap = d-ball cap fraction); tau_l = r^2;
//   - region: every lead row whose box distance to the tile's query bounding
//     box is <= sqrt(max tau_l), trimmed along the last dim to the cells the
//     ball around the box reaches -> a table of candidate spans (contiguous in
//     sorted order) in shared memory;
//   - scan: 32 candidates per chunk are loaded coalesced into shared memory and
//     broadcast; each lane appends candidates with fp32 sum (q-x)^2 <= tau_l to
//     its own list (16-bit (span, offset) codes, no top-k maintenance);
//   - certificate: the region covers the tau_l-ball of every lane, so the lane
//     is exact if >= need list entries lie strictly inside tau_l (3e-5 margin)
//     and the list did not overflow;
//   - epilogue per lane: bucket sort of the list on (d2/tau)^(d/2) (uniform for
//     uniform density), the buckets up to the one holding the need-th entry
//     (+1 for rounding safety) get float64 keys in the reference's operation
//     order (pyx:32-48) and an insertion sort; output slot = rank of
//     float32(d2_f64).  Two decided entries with equal float32 keys (ties /
//     sub-ulp near-ties) send the lane to the exact path.
// * anything the tile path cannot certify (overflow, sparse neighbourhood,
//   oversize tile, ties) is appended to a redo list that the warp-per-query
//   kernel finishes in a second launch -- same canonical answer either way.
#pragma once
#include "fg_knn_impl.cuh"

namespace fg {
namespace tile {

constexpr int kWarps = 4;          // warps per CTA
constexpr int kCap = 88;           // list entries per lane
constexpr int kSlack = 32;         // one chunk of overrun before the clamp
constexpr int kBkt = 32;           // epilogue buckets
constexpr int kHistStride = kBkt + 4;  // bytes per lane (bank spread)
constexpr int kMaxSpans = 384;     // candidate spans per tile
constexpr int kMaxSpanLen = 127;   // 7-bit offsets in the codes
constexpr float kAlpha = 1.12f;    // radius inflation over the density estimate
constexpr float kMargin = 1.0f + 1e-5f;
constexpr float kSlackCells = 1e-4f;
constexpr float kInf = __builtin_huge_valf();
constexpr int kMaxNeed = 40;       // host eligibility: k - 1 <= kMaxNeed

enum { TS_TILES, TS_CAND, TS_REDO, TS_TILE_FAIL, TS_COUNT };

struct TileArgs {
    const float4* sc;
    const int32_t* sid;
    const int32_t* bounds;
    const double* mins;
    const double* widths;
    int64_t total;     // n_bins^DB
    int nb, k, nblk;   // nblk = ceil(nb / 2)
    int bps;           // lead blocks per split = nblk^(DB-1)
    int n_blocks;      // S * bps
    int2* tiles;       // (block id, c_lo | c_hi << 8 | count << 16)
    int* ctr;          // [0] tiles, [1] tile cursor, [2] redo count
    int32_t* redo;     // sorted positions left for the warp-per-query kernel
    int32_t* out_idx;
    float* out_d2;
    unsigned long long* stats;
};

struct TileWarp {
    uint16_t code[(kCap + kSlack) * 32];  // [slot][lane] list entries
    float key[kCap * 32];                 // [slot][lane] epilogue keys
    uint8_t order[kCap * 32];             // [slot][lane] bucket-sorted entries
    uint8_t hist[32 * kHistStride];       // [lane][bucket]
    int32_t spS[kMaxSpans];               // span start (sorted position)
    uint16_t spE[kMaxSpans + 1];          // span flattened start (exclusive prefix)
    alignas(16) float sx[4][32];          // chunk coordinates, SoA
    alignas(16) uint32_t scode[32];       // chunk codes
};

__host__ __device__ constexpr size_t tile_smem_bytes() { return sizeof(TileWarp) * kWarps; }

// Lead block `b` of a split -> origin cells (last lead dim fastest).
template <int NL>
__device__ __forceinline__ void block_origin(int b, int nblk, int (&o)[NL > 0 ? NL : 1]) {
#pragma unroll
    for (int i = NL - 1; i >= 0; --i) {
        o[i] = 2 * (b % nblk);
        b /= nblk;
    }
}

// ---------------------------------------------------------------- tile list
// One warp per (split, lead block); lane c owns last-dim cell column c (nb <= 32).
template <int DB>
__global__ void __launch_bounds__(128) k_tiles(const TileArgs a) {
    constexpr int NL = DB - 1;
    const int lane = lane_id();
    const int blk = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (blk >= a.n_blocks) return;
    const int s = blk / a.bps;
    int o[NL > 0 ? NL : 1];
    block_origin<NL>(blk - s * a.bps, a.nblk, o);
    const int nb = a.nb;
    int col = 0;
    if (lane < nb) {
#pragma unroll
        for (int r = 0; r < (1 << NL); ++r) {
            int rowflat = 0;
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int j = o[i] + ((r >> (NL - 1 - i)) & 1);
                ok &= j < nb;
                rowflat = rowflat * nb + j;
            }
            if (ok) {
                const int64_t rc = (int64_t)s * a.total + (int64_t)rowflat * nb + lane;
                col += a.bounds[rc + 1] - a.bounds[rc];
            }
        }
    }
    const int P = warp_inclusive_scan(col);
    int start = 0, base = 0;
    while (start < nb) {  // warp-uniform greedy segmentation
        const unsigned bal = __ballot_sync(FG_FULL_MASK, lane >= start && lane < nb && P - base <= 32);
        const int end = bal ? 31 - __clz(bal) : start;  // P is non-decreasing: a prefix run
        const int pe = __shfl_sync(FG_FULL_MASK, P, end);
        const int cnt = pe - base;
        if (cnt > 0 && lane == 0) {
            const int t = atomicAdd(&a.ctr[0], 1);
            a.tiles[t] = make_int2(blk, start | (end << 8) | (min(cnt, 32767) << 16));
        }
        base = pe;
        start = end + 1;
    }
}

// ---------------------------------------------------------------- helpers
// Fraction of a DB-ball beyond a hyperplane at distance t*r from its centre.
template <int DB>
__device__ __forceinline__ float cap_frac(float t) {
    if (t >= 1.0f) return 0.0f;
    t = fmaxf(t, 0.0f);
    if (DB == 1) return 0.5f * (1.0f - t);
    if (DB == 2) return (acosf(t) - t * sqrtf(1.0f - t * t)) * 0.31830988f;
    if (DB == 3) return 0.25f * (1.0f - t) * (1.0f - t) * (2.0f + t);
    return 0.5f - (t * (5.0f - 2.0f * t * t) * sqrtf(1.0f - t * t) + 3.0f * asinf(t)) * 0.10610330f;
}

template <int DB>
__device__ __forceinline__ float unit_ball() {
    return DB == 1 ? 2.0f : DB == 2 ? 3.14159265f : DB == 3 ? 4.18879020f : 4.93480220f;
}

// (d2 / tau)^(DB/2): the share of a uniform ball inside radius sqrt(d2).
template <int DB>
__device__ __forceinline__ int bucket_of(float key, float inv_tau) {
    const float u = fminf(key * inv_tau, 1.0f);
    const float v = DB == 1 ? sqrtf(u) : DB == 2 ? u : DB == 3 ? u * sqrtf(u) : u * u;
    return min((int)(v * (float)kBkt), kBkt - 1);
}

// Query coordinates as packed fp32x2 registers: (q0,q1),(q2,q3) for one
// candidate, and every coordinate duplicated (qd,qd) for candidate pairs.
struct QP {
    unsigned long long lo, hi;
    unsigned long long dup[4];
};
__device__ __forceinline__ QP pack_q(const float4 q) {
    QP r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.lo) : "f"(q.x), "f"(q.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(r.hi) : "f"(q.z), "f"(q.w));
    asm("mov.b64 %0, {%1, %1};" : "=l"(r.dup[0]) : "f"(q.x));
    asm("mov.b64 %0, {%1, %1};" : "=l"(r.dup[1]) : "f"(q.y));
    asm("mov.b64 %0, {%1, %1};" : "=l"(r.dup[2]) : "f"(q.z));
    asm("mov.b64 %0, {%1, %1};" : "=l"(r.dup[3]) : "f"(q.w));
    return r;
}

// Four candidates of a chunk, SoA: x[dim] = (c_j, c_j+1), (c_j+2, c_j+3) pairs.
struct G4 {
    unsigned long long x[4][2];
};
__device__ __forceinline__ void load_g4(G4& g, uint32_t sx_addr, int j) {
#pragma unroll
    for (int d = 0; d < 4; ++d)
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                     : "=l"(g.x[d][0]), "=l"(g.x[d][1])
                     : "r"(sx_addr + d * 128 + j * 4));
}

// d2 of 4 candidates against the lane's query (packed over candidate pairs),
// predicated append of the passing candidates' codes to the lane's list.
__device__ __forceinline__ void eval_g4(const G4& g, const QP& q, float tau, uint32_t& ptr,
                                        uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    float d[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        unsigned long long t, acc;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(q.dup[0]), "l"(g.x[0][h]));
        asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(acc) : "l"(t));
#pragma unroll
        for (int dd = 1; dd < 4; ++dd) {
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t) : "l"(q.dup[dd]), "l"(g.x[dd][h]));
            asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(acc) : "l"(t), "l"(acc));
        }
        asm("mov.b64 {%0, %1}, %2;" : "=f"(d[2 * h]), "=f"(d[2 * h + 1]) : "l"(acc));
    }
    const uint32_t cs[4] = {c0, c1, c2, c3};
#pragma unroll
    for (int i = 0; i < 4; ++i)
        asm volatile(
            "{ .reg .pred p; setp.le.f32 p, %1, %2; @p st.shared.u16 [%0], %3; "
            "@p add.u32 %0, %0, 64; }"
            : "+r"(ptr)
            : "f"(d[i]), "f"(tau), "r"(cs[i]));
}

// fp32 sum (q-c)^2 of one candidate, packed: ((q0-c0)^2 + (q2-c2)^2) +
// ((q1-c1)^2 + (q3-c3)^2).  Any fp32 order is within ~1e-6 of the float64
// value, far inside every 1e-5 margin of the certificate.
__device__ __forceinline__ float d2_f32(const QP& q, const float4 c) {
    unsigned long long c01, c23, t01, t23, acc;
    asm("mov.b64 %0, {%1, %2};" : "=l"(c01) : "f"(c.x), "f"(c.y));
    asm("mov.b64 %0, {%1, %2};" : "=l"(c23) : "f"(c.z), "f"(c.w));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t01) : "l"(q.lo), "l"(c01));
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t23) : "l"(q.hi), "l"(c23));
    asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(acc) : "l"(t01));
    asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(acc) : "l"(t23), "l"(acc));
    float a0, a1;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
    return a0 + a1;
}

__device__ __forceinline__ unsigned f2o(float f) { return float_to_ordered(f); }

__device__ __forceinline__ float warp_min_f(float v) {
    return ordered_to_float(__reduce_min_sync(FG_FULL_MASK, f2o(v)));
}
__device__ __forceinline__ float warp_max_f(float v) {
    return ordered_to_float(__reduce_max_sync(FG_FULL_MASK, f2o(v)));
}

__device__ __forceinline__ void push_redo(const TileArgs& a, bool redo, int32_t p) {
    const unsigned bal = __ballot_sync(FG_FULL_MASK, redo);
    if (!bal) return;
    int base = 0;
    if (lane_id() == 0) base = atomicAdd(&a.ctr[2], __popc(bal));
    base = __shfl_sync(FG_FULL_MASK, base, 0);
    if (redo) a.redo[base + __popc(bal & lanemask_lt())] = p;
}

// ---------------------------------------------------------------- search
template <int DB>
__global__ void __launch_bounds__(kWarps * 32, 2) k_tile_search(const __grid_constant__ TileArgs a) {
    constexpr int NL = DB - 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileWarp& W = reinterpret_cast<TileWarp*>(smem_raw)[threadIdx.x >> 5];
    const int lane = lane_id();
    const int nb = a.nb;
    const int need = a.k - 1;
    const int n_tiles = a.ctr[0];
    unsigned long long st_cand = 0, st_tiles = 0, st_redo = 0, st_fail = 0;

    for (;;) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&a.ctr[1], 1);
        t = __shfl_sync(FG_FULL_MASK, t, 0);
        if (t >= n_tiles) break;
        ++st_tiles;
        const int2 tl = a.tiles[t];
        const int blk = tl.x;
        const int c_lo = tl.y & 255, c_hi = (tl.y >> 8) & 255, cnt = tl.y >> 16;
        const int s = blk / a.bps;
        int o[NL > 0 ? NL : 1];
        block_origin<NL>(blk - s * a.bps, a.nblk, o);
        const int64_t cbase = (int64_t)s * a.total;

        // ---- the tile's points: rows of the block, cells [c_lo, c_hi]
        int32_t rS = 0, rL = 0;
        if (lane < (1 << NL)) {
            int rowflat = 0;
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int j = o[i] + ((lane >> (NL - 1 - i)) & 1);
                ok &= j < nb;
                rowflat = rowflat * nb + j;
            }
            if (ok) {
                const int64_t rc = cbase + (int64_t)rowflat * nb;
                rS = a.bounds[rc + c_lo];
                rL = a.bounds[rc + c_hi + 1] - rS;
            }
        }
        const int32_t rIncl = warp_inclusive_scan(rL);
        if (cnt > 32) {  // oversize tile (one column holds > 32 points): exact path
            ++st_fail;
            for (int r = 0; r < (1 << NL); ++r) {
                const int32_t S = __shfl_sync(FG_FULL_MASK, rS, r);
                const int32_t L = __shfl_sync(FG_FULL_MASK, rL, r);
                for (int i0 = 0; i0 < L; i0 += 32) {
                    push_redo(a, i0 + lane < L, S + i0 + lane);
                    st_redo += (i0 + lane < L) ? 1 : 0;
                }
            }
            continue;
        }
        int32_t p = -1;
#pragma unroll
        for (int r = 0; r < (1 << NL); ++r) {
            const int32_t S = __shfl_sync(FG_FULL_MASK, rS, r);
            const int32_t I = __shfl_sync(FG_FULL_MASK, rIncl, r);
            const int32_t L = __shfl_sync(FG_FULL_MASK, rL, r);
            if (lane >= I - L && lane < I) p = S + (lane - (I - L));
        }
        const bool active = p >= 0;
        float4 q = make_float4(0.f, 0.f, 0.f, 0.f);
        if (active) q = a.sc[p];
        const float qa[4] = {q.x, q.y, q.z, q.w};
        float mn[DB], w[DB], invw[DB], qc[DB], lo[DB], hi[DB];
#pragma unroll
        for (int i = 0; i < DB; ++i) {
            mn[i] = (float)a.mins[(int64_t)s * DB + i];
            w[i] = (float)a.widths[(int64_t)s * DB + i];
            invw[i] = __frcp_rn(w[i]);
            qc[i] = (qa[i] - mn[i]) * invw[i];
            lo[i] = warp_min_f(active ? qc[i] : kInf);
            hi[i] = warp_max_f(active ? qc[i] : -kInf);
        }

        // ---- density of the block's neighbourhood -> r_k
        int dl[NL > 0 ? NL : 1], dn[NL > 0 ? NL : 1];
        int drows = 1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            dl[i] = max(o[i] - 1, 0);
            dn[i] = min(o[i] + 2, nb - 1) - dl[i] + 1;
            drows *= dn[i];
        }
        const int dA = max(c_lo - 1, 0), dB = min(c_hi + 1, nb - 1);
        int dcnt = 0;
        for (int r = lane; r < drows; r += 32) {
            int rr = r, rowflat = 0, jj[NL > 0 ? NL : 1];
#pragma unroll
            for (int i = NL - 1; i >= 0; --i) {
                jj[i] = dl[i] + rr % dn[i];
                rr /= dn[i];
            }
#pragma unroll
            for (int i = 0; i < NL; ++i) rowflat = rowflat * nb + jj[i];
            const int64_t rc = cbase + (int64_t)rowflat * nb;
            dcnt += a.bounds[rc + dB + 1] - a.bounds[rc + dA];
        }
        dcnt = __reduce_add_sync(FG_FULL_MASK, dcnt);
        bool tile_fail = dcnt < 2 * need + 2;
        float vol = (float)(drows * (dB - dA + 1));
#pragma unroll
        for (int i = 0; i < DB; ++i) vol *= w[i];
        const float rk = exp2f(__log2f((float)need * vol / ((float)dcnt * unit_ball<DB>())) *
                               (1.0f / (float)DB));
        // per-lane radius corrected for the part of the ball outside the grid
        float rad = kAlpha * rk;
#pragma unroll 1
        for (int it = 0; it < 3; ++it) {
            float f = 1.0f;
#pragma unroll
            for (int i = 0; i < DB; ++i) {
                const float h0 = qa[i] - mn[i];
                const float h1 = (float)nb * w[i] - h0;
                f *= 1.0f - cap_frac<DB>(h0 / rad) - cap_frac<DB>(h1 / rad);
            }
            f = fmaxf(f, 0.05f);
            rad = kAlpha * rk * exp2f(__log2f(f) * (-1.0f / (float)DB));
        }
        const float tau = active ? rad * rad : -1.0f;  // inactive lanes append nothing
        const float tau_max = warp_max_f(tau);
        tile_fail |= !(tau_max < kInf);

        // ---- region -> span table
        const float rr_max = sqrtf(tau_max) * kMargin;
        int L[NL > 0 ? NL : 1], N[NL > 0 ? NL : 1];
        float inv[NL > 0 ? NL : 1];
        int nrows = 1;
#pragma unroll
        for (int i = 0; i < NL; ++i) {
            const float rc = rr_max * invw[i] + kSlackCells;
            L[i] = (int)fmaxf(floorf(lo[i] - rc), 0.0f);
            N[i] = (int)fminf(floorf(hi[i] + rc), (float)(nb - 1)) - L[i] + 1;
            inv[i] = __frcp_rn((float)N[i]);
            nrows *= N[i];
        }
        int nsp = 0, T = 0;
        bool bad = tile_fail;
        for (int rb = 0; rb < nrows && !bad; rb += 32) {
            const int r = rb + lane;
            int32_t S = 0, Ln = 0;
            if (r < nrows) {
                int jd[NL > 0 ? NL : 1];
                search::decode_row<NL>(r, L, N, inv, jd);
                int rowflat = 0;
                float bd2 = 0.0f;
#pragma unroll
                for (int i = 0; i < NL; ++i) {
                    rowflat = rowflat * nb + jd[i];
                    const float fj = (float)jd[i];
                    float g = fmaxf(fmaxf(fj - hi[i], lo[i] - (fj + 1.0f)) - kSlackCells, 0.0f) * w[i];
                    bd2 = fmaf(g, g, bd2);
                }
                const float rem = tau_max - bd2;
                if (rem >= 0.0f) {
                    const float rc = sqrtf(rem) * invw[NL] * kMargin + kSlackCells;
                    const int ca = (int)fmaxf(floorf(lo[NL] - rc), 0.0f);
                    const int cb = (int)fminf(floorf(hi[NL] + rc), (float)(nb - 1));
                    if (ca <= cb) {
                        const int64_t rc0 = cbase + (int64_t)rowflat * nb;
                        S = a.bounds[rc0 + ca];
                        Ln = a.bounds[rc0 + cb + 1] - S;
                    }
                }
            }
            const unsigned ne = __ballot_sync(FG_FULL_MASK, Ln > 0);
            bad |= __any_sync(FG_FULL_MASK, Ln > kMaxSpanLen);
            const int32_t incl = warp_inclusive_scan(Ln);
            const int tot = __shfl_sync(FG_FULL_MASK, incl, 31);
            const int g = nsp + __popc(ne & lanemask_lt());
            bad |= nsp + __popc(ne) > kMaxSpans || T + tot > 65535 - 64;
            if (!bad && Ln > 0) {
                W.spS[g] = S;
                W.spE[g] = (uint16_t)(T + incl - Ln);
            }
            nsp += __popc(ne);
            T += tot;
        }
        if (bad) {
            ++st_fail;
            push_redo(a, active, p);
            st_redo += active ? 1 : 0;
            __syncwarp();
            continue;
        }
        if (lane == 0) W.spE[nsp] = (uint16_t)T;
        __syncwarp();
        st_cand += T;

        // ---- scan: 32 candidates per chunk, broadcast to every lane
        const QP qv = pack_q(q);
        const uint32_t lbase = (uint32_t)__cvta_generic_to_shared(&W.code[lane]);
        const uint32_t llim = lbase + kCap * 64;
        const uint32_t sx_addr = (uint32_t)__cvta_generic_to_shared(&W.sx[0][0]);
        uint32_t ptr = lbase;
        bool overflow = false;
        int s0 = 0;
        for (int f0 = 0; f0 < T; f0 += 32) {
            const int f = f0 + lane;
            const int si = s0 + lane;
            const int st = si < nsp ? W.spE[si] : 0x7fffffff;
            const unsigned starts = __reduce_or_sync(
                FG_FULL_MASK, (lane > 0 && st > f0 && st < f0 + 32) ? 1u << (st - f0) : 0u);
            const int g = s0 + __popc(starts & ((2u << lane) - 1u));
            float4 c = make_float4(kInf, kInf, kInf, kInf);
            uint32_t code = 0;
            if (f < T) {
                const int off = f - W.spE[g];
                c = a.sc[W.spS[g] + off];
                code = (uint32_t)((g << 7) | off);
            }
            W.sx[0][lane] = c.x;
            W.sx[1][lane] = c.y;
            W.sx[2][lane] = c.z;
            W.sx[3][lane] = c.w;
            W.scode[lane] = code;
            s0 = __shfl_sync(FG_FULL_MASK, g, 31);
            if (s0 + 1 < nsp && W.spE[s0 + 1] == f0 + 32) ++s0;
            __syncwarp();
            uint32_t cd[32];  // the chunk's codes (uniform), in registers
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint4 v = reinterpret_cast<const uint4*>(W.scode)[j];
                cd[4 * j] = v.x; cd[4 * j + 1] = v.y; cd[4 * j + 2] = v.z; cd[4 * j + 3] = v.w;
            }
            // software pipeline: the next group's loads precede this group's stores
            G4 gb[2];
            load_g4(gb[0], sx_addr, 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j + 1 < 8) load_g4(gb[(j + 1) & 1], sx_addr, 4 * (j + 1));
                eval_g4(gb[j & 1], qv, tau, ptr, cd[4 * j], cd[4 * j + 1], cd[4 * j + 2],
                        cd[4 * j + 3]);
            }
            if (ptr > llim) {
                overflow = true;
                ptr = llim;
            }
            __syncwarp();
        }
        asm volatile("" ::: "memory");  // list stores (inline asm) before the epilogue reads

        // ---- epilogue (per lane)
        const int m = (int)(ptr - lbase) >> 6;
        bool ok = active && !overflow;
        const float inner = tau * (1.0f - 3e-5f);
        const float inv_tau = tau > 0.0f ? 1.0f / tau : 0.0f;
        uint8_t* hist = &W.hist[lane * kHistStride];
#pragma unroll
        for (int b = 0; b < kBkt; b += 4) *reinterpret_cast<uint32_t*>(hist + b) = 0u;
        int n_in = 0;
        const int m_run = ok ? m : 0;
        for (int e = 0; e < m_run; ++e) {
            const uint16_t cd = W.code[e * 32 + lane];
            const int32_t cpos = W.spS[cd >> 7] + (cd & 127);
            float key = kInf;
            if (cpos != p) {
                key = d2_f32(qv, a.sc[cpos]);
                n_in += key < inner ? 1 : 0;
                hist[bucket_of<DB>(key, inv_tau)]++;
            }
            W.key[e * 32 + lane] = key;
        }
        ok &= n_in >= need;
        // buckets up to the one holding the need-th entry, plus one
        int M = 0, bstar = kBkt;
        if (ok) {
            int cum = 0;
            for (int b = 0; b < kBkt; ++b) {
                const int h = hist[b];
                hist[b] = (uint8_t)cum;
                cum += h;
                if (bstar == kBkt && cum >= need) bstar = b;
                if (b <= bstar + 1) M = cum;
            }
            for (int e = 0; e < m; ++e) {
                const float key = W.key[e * 32 + lane];
                if (key < kInf) {
                    const int b = bucket_of<DB>(key, inv_tau);
                    if (b <= bstar + 1) {
                        const int sl = hist[b];
                        hist[b] = (uint8_t)(sl + 1);
                        W.order[sl * 32 + lane] = (uint8_t)e;
                    }
                }
            }
            // float64 keys for the decided range, then insertion sort
            for (int sl = 0; sl < M; ++sl) {
                const int e = W.order[sl * 32 + lane];
                const uint16_t cd = W.code[e * 32 + lane];
                const float4 c = a.sc[W.spS[cd >> 7] + (cd & 127)];
                const float cq[4] = {c.x, c.y, c.z, c.w};
                W.key[e * 32 + lane] = __double2float_rn(exact_d2<DB>(qa, cq, DB));
            }
            for (int sl = 1; sl < M; ++sl) {
                const int x = W.order[sl * 32 + lane];
                const float kx = W.key[x * 32 + lane];
                int t2 = sl - 1;
                int y = W.order[t2 * 32 + lane];
                while (W.key[y * 32 + lane] > kx) {
                    W.order[(t2 + 1) * 32 + lane] = (uint8_t)y;
                    if (--t2 < 0) break;
                    y = W.order[t2 * 32 + lane];
                }
                W.order[(t2 + 1) * 32 + lane] = (uint8_t)x;
            }
            bool amb = false;
            float prev = W.key[W.order[lane] * 32 + lane];
            for (int sl = 1; sl < min(M, need + 1); ++sl) {
                const float kk = W.key[W.order[sl * 32 + lane] * 32 + lane];
                amb |= kk == prev;
                prev = kk;
            }
            ok &= !amb;
        }
        // ---- output rows (sorted), or the exact path
        if (ok) {
            const int32_t qid = a.sid[p];
            int32_t* oi = a.out_idx + (int64_t)qid * a.k;
            float* od = a.out_d2 + (int64_t)qid * a.k;
            oi[0] = qid;
            od[0] = 0.0f;
            for (int sl = 0; sl < need; ++sl) {
                const int e = W.order[sl * 32 + lane];
                const uint16_t cd = W.code[e * 32 + lane];
                oi[1 + sl] = a.sid[W.spS[cd >> 7] + (cd & 127)];
                od[1 + sl] = W.key[e * 32 + lane];
            }
        }
        const bool redo = active && !ok;
        push_redo(a, redo, p);
        st_redo += redo ? 1 : 0;
        __syncwarp();
    }
    if (a.stats) {
        st_redo = __reduce_add_sync(FG_FULL_MASK, (unsigned)st_redo);
        if (lane == 0) {
            atomicAdd(&a.stats[TS_TILES], st_tiles);
            atomicAdd(&a.stats[TS_CAND], st_cand);
            atomicAdd(&a.stats[TS_REDO], st_redo);
            atomicAdd(&a.stats[TS_TILE_FAIL], st_fail);
        }
    }
}

}  // namespace tile
}  // namespace fg
