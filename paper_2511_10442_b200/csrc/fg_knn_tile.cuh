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
#include <type_traits>

#include "fg_knn_impl.cuh"

namespace fg {
namespace tile {

constexpr int kWarps = 4;          // warps per CTA (4 CTAs per SM: 16 warps)
constexpr int kCap = 88;           // list entries per lane
constexpr int kSlack = 16;         // half a chunk of overrun before the clamp
constexpr int kStride = kCap + kSlack + 2;  // u16 per lane list: 53 words, odd -> bank spread
#ifndef FG_TILE_CTAS
#define FG_TILE_CTAS 4
#endif
constexpr int kCtasPerSm = FG_TILE_CTAS;
constexpr int kBkt = 128;          // epilogue buckets (4 per lane)
constexpr int kMaxSpans = 320;     // candidate spans per tile
constexpr int kMaxSpanLen = 127;   // 7-bit offsets in the codes
#ifndef FG_TILE_ALPHA
#define FG_TILE_ALPHA 1.10f
#endif
#ifndef FG_RADIUS_ITERS
#define FG_RADIUS_ITERS 2
#endif
constexpr float kAlpha = FG_TILE_ALPHA;  // radius inflation over the density estimate
constexpr float kMargin = 1.0f + 1e-5f;
constexpr float kSlackCells = 1e-4f;
constexpr float kInf = __builtin_huge_valf();
constexpr int kMaxNeed = 40;       // host eligibility: k - 1 <= kMaxNeed

enum { TS_TILES, TS_CAND, TS_REDO, TS_TILE_FAIL, TS_EXPANDED, TS_EVAL, TS_COUNT };

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
    int* ctr;          // [0] tiles, [1] tile cursor, [2] redo count, [4] points in oversize columns
    int64_t n;         // points (all splits)
    int32_t* redo;     // sorted positions left for the warp-per-query kernel
    int32_t* out_idx;
    float* out_d2;
    unsigned long long* stats;
    // split epilogue (non-null): the scan kernel writes each query's candidate
    // list (sorted positions, kCap per query) and (tau, m); k_tile_finish sorts
    int32_t* lists;
    float2* meta;
    // high-dimensional path (fg_knn_hd.cuh): search copies of sc / sid with the
    // points of dense cells in Morton order of their sub-cell position (null:
    // the binning's order is used as is)
    float4* sc2;
    int32_t* sid2;
    int32_t* dense;
    // hd path: points per tile (1..32; tiles[t] = (block, first point in block order))
    uint8_t* tcnt;
    // hd path dispatch order (widest query boxes first): per-tile cost bucket,
    // bucket counts / cursors (2 x 64), the order (null: tile order)
    uint8_t* tkey;
    int* hist;
    int32_t* order;
    // hd path, d <= 4: bounding box (lo, hi) of every 32 sorted positions of
    // the search's coordinates (2 float4 per block; null: not used)
    float4* boxes;
    // hd path as the clustered-data fallback of the d <= 4 tile path: run only
    // when *gate * 4 > n (the tile kernels declined the data); null: always
    const int* gate;
    // host-mapped flag: the scan kernel records whether it declined the data,
    // so the next call launches the (gated) fallback only when the data of
    // the previous call was clustered (either way the answer is the same)
    volatile int* hint;
};

// The hd kernels' gate (see TileArgs::gate).
__device__ __forceinline__ bool gated_off(const TileArgs& a) {
    return a.gate && (int64_t)*a.gate * 4 <= a.n;
}

// Per-warp shared memory of the scan.
struct ScanWarp {
    uint16_t code[32 * kStride];          // [lane][slot] per-lane candidate lists
    int32_t spS[kMaxSpans];               // span start (sorted position)
    uint16_t spE[kMaxSpans + 1];          // span flattened start (exclusive prefix)
    alignas(16) float sx[4][64];          // candidate ring (2 chunks), SoA (centred when expanded)
    alignas(16) float sn[64];             // expanded mode: |c - centre|^2 (ring)
    alignas(16) uint16_t scode[64];       // ring codes
};
// ... plus the epilogue staging when the scan kernel finishes its own queries
// (FG_KNN_FUSED_EPI, a diagnostics variant).
struct TileWarp : ScanWarp {
    float skey[kCap];                     // epilogue staging of one query: keys
    int32_t sid[kCap];                    //   and original ids, in bucket order
    alignas(16) float okey[kCap + 4];     //   final row: slot 0 = self, then by key
    alignas(16) int32_t oid[kCap + 4];
    alignas(16) uint32_t bcnt[kBkt + 4];  //   bucket counts -> starts
};

#ifndef FG_SCAN_CTAS
#define FG_SCAN_CTAS 5
#endif
constexpr int kScanCtasPerSm = FG_SCAN_CTAS;  // the split-epilogue scan kernel

template <bool SPLIT>
__host__ __device__ constexpr size_t tile_smem_bytes() {
    return (SPLIT ? sizeof(ScanWarp) : sizeof(TileWarp)) * kWarps;
}
static_assert(tile_smem_bytes<false>() * kCtasPerSm + 1024 * kCtasPerSm <= 233472,
              "k_tile_search: CTAs per SM do not fit in shared memory");
static_assert(tile_smem_bytes<true>() * kScanCtasPerSm + 1024 * kScanCtasPerSm <= 233472,
              "k_tile_search (split): CTAs per SM do not fit in shared memory");

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
    // warp-uniform greedy segmentation (P is non-decreasing: each segment is a
    // prefix run of the remaining columns), tiles staged in registers and
    // claimed with one atomic per block
    int start = 0, base = 0, nt = 0;
    int2 mine = make_int2(0, 0);
    while (start < nb) {
        const unsigned bal = __ballot_sync(FG_FULL_MASK, lane >= start && lane < nb && P - base <= 32);
        const int end = bal ? 31 - __clz(bal) : start;
        const int pe = __shfl_sync(FG_FULL_MASK, P, end);
        const int cnt = pe - base;
        if (cnt > 0) {
            if (lane == nt) mine = make_int2(blk, start | (end << 8) | (min(cnt, 32767) << 16));
            ++nt;
            if (cnt > 32 && lane == 0) atomicAdd(&a.ctr[4], cnt);  // clustered-data detector
        }
        base = pe;
        start = end + 1;
    }
    int t0 = 0;
    if (lane == 0 && nt > 0) t0 = atomicAdd(&a.ctr[0], nt);
    t0 = __shfl_sync(FG_FULL_MASK, t0, 0);
    if (lane < nt) a.tiles[t0 + lane] = mine;
}

// More than a quarter of the points in columns too dense for a tile: the data
// is clustered at the cell scale and the radius hint fails there; the tile
// kernels step aside and the warp-per-query kernel takes every query in
// sorted order (decided on the device, no host synchronisation).
__device__ __forceinline__ bool tiles_declined(const TileArgs& a) {
    return (int64_t)a.ctr[4] * 4 > a.n;
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

// Predicated append of up to four candidate codes (d <= thr) to the lane's
// list (one asm block: no register copies of the list pointer in between).
__device__ __forceinline__ void append4(uint32_t& ptr, const float (&d)[4], float thr, uint32_t c0,
                                        uint32_t c1, uint32_t c2, uint32_t c3) {
    asm volatile(
        "{ .reg .pred p0, p1, p2, p3;\n\t"
        "setp.le.f32 p0, %1, %5;\n\t"
        "setp.le.f32 p1, %2, %5;\n\t"
        "setp.le.f32 p2, %3, %5;\n\t"
        "setp.le.f32 p3, %4, %5;\n\t"
        "@p0 st.shared.u16 [%0], %6;\n\t"
        "@p0 add.u32 %0, %0, 2;\n\t"
        "@p1 st.shared.u16 [%0], %7;\n\t"
        "@p1 add.u32 %0, %0, 2;\n\t"
        "@p2 st.shared.u16 [%0], %8;\n\t"
        "@p2 add.u32 %0, %0, 2;\n\t"
        "@p3 st.shared.u16 [%0], %9;\n\t"
        "@p3 add.u32 %0, %0, 2; }"
        : "+r"(ptr)
        : "f"(d[0]), "f"(d[1]), "f"(d[2]), "f"(d[3]), "f"(thr), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
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
                     : "r"(sx_addr + d * 256 + j * 4));
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
    append4(ptr, d, tau, c0, c1, c2, c3);
}

// Expanded form around the tile centre: d2 = |q'|^2 + |c'|^2 - 2 q'.c' with
// q' = q - centre, c' = c - centre (FADD2 + 4 FFMA2 per candidate pair).  Used
// only when its rounding error, <= 12u (|q'| + |c'|)^2 + 2u (|q'| + |c'|) |q-c|,
// stays below 2.5e-5 tau of every lane (checked per tile); else the direct form.
struct QX {
    unsigned long long sq;      // (|q'|^2, |q'|^2)
    unsigned long long m2q[4];  // (-2 q'_d, -2 q'_d)
    float tau_x;                // tau - |q'|^2: |c'|^2 - 2 q'.c' is compared with it
};
struct G4X {
    unsigned long long x[4][2];
    unsigned long long n[2];
};
__device__ __forceinline__ void load_g4x(G4X& g, uint32_t sx_addr, int j) {
#pragma unroll
    for (int d = 0; d < 4; ++d)
        asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                     : "=l"(g.x[d][0]), "=l"(g.x[d][1])
                     : "r"(sx_addr + d * 256 + j * 4));
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];"
                 : "=l"(g.n[0]), "=l"(g.n[1])
                 : "r"(sx_addr + 4 * 256 + j * 4));
}
__device__ __forceinline__ void eval_g4x(const G4X& g, const QX& q, float tau_x, uint32_t& ptr,
                                         uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    float d[4];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // |c'|^2 - 2 q'.c' for a candidate pair: 4 FFMA2
        unsigned long long acc = g.n[h];
#pragma unroll
        for (int dd = 0; dd < 4; ++dd)
            asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(acc) : "l"(g.x[dd][h]), "l"(q.m2q[dd]), "l"(acc));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(d[2 * h]), "=f"(d[2 * h + 1]) : "l"(acc));
    }
    append4(ptr, d, tau_x, c0, c1, c2, c3);
}

__device__ __forceinline__ unsigned long long pack2(float x) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}

// Stream the tile's candidates in 32-candidate chunks (coalesced loads into
// shared memory, then broadcast) and append each lane's passing codes.
template <bool EXP>
__device__ __forceinline__ void scan_tile(ScanWarp& W, const float4* __restrict__ sc, int T, int nsp,
                                          const QP& qv, const QX& qx, const float4 cen, float tau,
                                          uint32_t& ptr, bool& overflow, uint32_t llim) {
    const int lane = lane_id();
    const uint32_t sx_addr = (uint32_t)__cvta_generic_to_shared(&W.sx[0][0]);
    // chunk c+1's candidate is loaded (global) while chunk c is evaluated
    int s0 = 0;
    auto fetch = [&](int f0, float4& c, uint32_t& code, bool& live) {
        const int f = f0 + lane;
        const int si = s0 + lane;
        const int st = si < nsp ? W.spE[si] : 0x7fffffff;
        const unsigned starts = __reduce_or_sync(
            FG_FULL_MASK, (lane > 0 && st > f0 && st < f0 + 32) ? 1u << (st - f0) : 0u);
        const int g = s0 + __popc(starts & ((2u << lane) - 1u));
        live = f < T;
        code = 0;
        if (live) {
            const int off = f - W.spE[g];
            c = sc[W.spS[g] + off];
            code = (uint32_t)((g << 7) | off);
        }
        s0 = __shfl_sync(FG_FULL_MASK, g, 31);
        if (s0 + 1 < nsp && W.spE[s0 + 1] == f0 + 32) ++s0;
    };
    float4 cn = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t coden = 0;
    bool liven = false;
    if (T > 0) fetch(0, cn, coden, liven);
    for (int f0 = 0; f0 < T; f0 += 32) {
        float4 c = cn;
        const uint32_t code = coden;
        const bool live = liven;
        if (f0 + 32 < T) fetch(f0 + 32, cn, coden, liven);
        float nn = kInf;
        if (!live) {
            c = EXP ? make_float4(0.f, 0.f, 0.f, 0.f) : make_float4(kInf, kInf, kInf, kInf);
        } else if (EXP) {
            c.x -= cen.x; c.y -= cen.y; c.z -= cen.z; c.w -= cen.w;
            nn = fmaf(c.w, c.w, fmaf(c.z, c.z, fmaf(c.y, c.y, c.x * c.x)));
        }
        W.sx[0][lane] = c.x;
        W.sx[1][lane] = c.y;
        W.sx[2][lane] = c.z;
        W.sx[3][lane] = c.w;
        if (EXP) W.sn[lane] = nn;
        W.scode[lane] = (uint16_t)code;
        __syncwarp();
        // software pipeline: the next group's loads precede this group's stores
        if (EXP) {
            uint32_t cd[32];  // the chunk's codes (uniform), in registers
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 v = reinterpret_cast<const uint4*>(W.scode)[j];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    cd[8 * j + 2 * h] = w4[h];
                    cd[8 * j + 2 * h + 1] = w4[h] >> 16;
                }
            }
            G4X gb[2];
            load_g4x(gb[0], sx_addr, 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j + 1 < 8) load_g4x(gb[(j + 1) & 1], sx_addr, 4 * (j + 1));
                eval_g4x(gb[j & 1], qx, qx.tau_x, ptr, cd[4 * j], cd[4 * j + 1], cd[4 * j + 2],
                         cd[4 * j + 3]);
                if (j == 3 && ptr > llim) {  // clamp every 16 candidates (kSlack)
                    overflow = true;
                    ptr = llim;
                }
            }
        } else {
            // direct form: 4 floats per candidate from shared memory (the scan is
            // bound by the shared-memory pipe; the expanded form reads 5); the
            // 16-bit codes come in 4 vector loads, odd ones shifted down
            uint32_t cd[32];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint4 v = reinterpret_cast<const uint4*>(W.scode)[j];
                const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    cd[8 * j + 2 * h] = w4[h];  // st.shared.u16 keeps the low half
                    cd[8 * j + 2 * h + 1] = w4[h] >> 16;
                }
            }
            G4 gb[2];
            load_g4(gb[0], sx_addr, 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j + 1 < 8) load_g4(gb[(j + 1) & 1], sx_addr, 4 * (j + 1));
                eval_g4(gb[j & 1], qv, tau, ptr, cd[4 * j], cd[4 * j + 1], cd[4 * j + 2],
                        cd[4 * j + 3]);
                if (j == 3 && ptr > llim) {
                    overflow = true;
                    ptr = llim;
                }
            }
        }
        if (ptr > llim) {
            overflow = true;
            ptr = llim;
        }
        __syncwarp();
    }
}

// Direct-form scan with a per-candidate filter: a candidate farther than
// sqrt(tau_max) from the tile's query bounding box cannot enter any lane's list
// (about half of the region's candidates at north_star: the region is built
// at cell granularity).  Fetched chunks are compacted into a 64-entry ring and
// evaluated 32 at a time, so the broadcast loop only sees useful candidates.
template <bool EXP>
__device__ __forceinline__ void scan_tile_filtered(ScanWarp& W, const float4* __restrict__ sc, int T,
                                                   int nsp, const QP& qv, const QX& qx,
                                                   const float4 cen, float tau,
                                                   const float4 blo, const float4 bhi, float thr,
                                                   uint32_t& ptr, bool& overflow, uint32_t llim,
                                                   unsigned long long& n_eval) {
    const int lane = lane_id();
    const uint32_t sx_addr = (uint32_t)__cvta_generic_to_shared(&W.sx[0][0]);
    int s0 = 0;
    auto fetch = [&](int f0, float4& c, uint32_t& code, bool& live) {
        const int f = f0 + lane;
        const int si = s0 + lane;
        const int st = si < nsp ? W.spE[si] : 0x7fffffff;
        const unsigned starts = __reduce_or_sync(
            FG_FULL_MASK, (lane > 0 && st > f0 && st < f0 + 32) ? 1u << (st - f0) : 0u);
        const int g = s0 + __popc(starts & ((2u << lane) - 1u));
        live = f < T;
        code = 0;
        if (live) {
            const int off = f - W.spE[g];
            c = sc[W.spS[g] + off];
            code = (uint32_t)((g << 7) | off);
        }
        s0 = __shfl_sync(FG_FULL_MASK, g, 31);
        if (s0 + 1 < nsp && W.spE[s0 + 1] == f0 + 32) ++s0;
    };
    float4 cn = make_float4(0.f, 0.f, 0.f, 0.f);
    uint32_t coden = 0;
    bool liven = false;
    int fpos = 0;
    if (T > 0) fetch(0, cn, coden, liven);
    int head = 0, filled = 0;
    for (;;) {
        while (filled < 32 && fpos < T) {  // fill the ring with useful candidates
            const float4 c = cn;
            const uint32_t code = coden;
            const bool live = liven;
            fpos += 32;
            if (fpos < T) fetch(fpos, cn, coden, liven);  // next raw chunk in flight
            float g = fmaxf(fmaxf(blo.x - c.x, c.x - bhi.x), 0.0f);
            float dd = g * g;
            g = fmaxf(fmaxf(blo.y - c.y, c.y - bhi.y), 0.0f);
            dd = fmaf(g, g, dd);
            g = fmaxf(fmaxf(blo.z - c.z, c.z - bhi.z), 0.0f);
            dd = fmaf(g, g, dd);
            g = fmaxf(fmaxf(blo.w - c.w, c.w - bhi.w), 0.0f);
            dd = fmaf(g, g, dd);
            const bool useful = live && dd <= thr;
            const unsigned bal = __ballot_sync(FG_FULL_MASK, useful);
            if (useful) {
                const int slot = (head + filled + __popc(bal & lanemask_lt())) & 63;
                if (EXP) {  // centred on the tile box, with |c'|^2
                    const float4 cc = make_float4(c.x - cen.x, c.y - cen.y, c.z - cen.z, c.w - cen.w);
                    W.sx[0][slot] = cc.x;
                    W.sx[1][slot] = cc.y;
                    W.sx[2][slot] = cc.z;
                    W.sx[3][slot] = cc.w;
                    W.sn[slot] = fmaf(cc.w, cc.w, fmaf(cc.z, cc.z, fmaf(cc.y, cc.y, cc.x * cc.x)));
                } else {
                    W.sx[0][slot] = c.x;
                    W.sx[1][slot] = c.y;
                    W.sx[2][slot] = c.z;
                    W.sx[3][slot] = c.w;
                }
                W.scode[slot] = (uint16_t)code;
            }
            filled += __popc(bal);
        }
        if (filled == 0) break;
        if (filled < 32 && lane >= filled) {  // last round: pad with far-away sentinels
            const int slot = (head + lane) & 63;
            if (EXP) {
                W.sx[0][slot] = 0.f; W.sx[1][slot] = 0.f; W.sx[2][slot] = 0.f; W.sx[3][slot] = 0.f;
                W.sn[slot] = kInf;
            } else {
                W.sx[0][slot] = kInf; W.sx[1][slot] = kInf; W.sx[2][slot] = kInf; W.sx[3][slot] = kInf;
            }
        }
        __syncwarp();
        n_eval += 32;
        const uint32_t base = sx_addr + head * 4;
        uint32_t cd[32];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 v = reinterpret_cast<const uint4*>(&W.scode[head])[j];
            const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                cd[8 * j + 2 * h] = w4[h];  // st.shared.u16 keeps the low half
                cd[8 * j + 2 * h + 1] = w4[h] >> 16;
            }
        }
        if (EXP) {  // |c'|^2 - 2 q'.c' against tau - |q'|^2: 4 FFMA2 per candidate pair
            G4X gb[2];
            load_g4x(gb[0], base, 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j + 1 < 8) load_g4x(gb[(j + 1) & 1], base, 4 * (j + 1));
                eval_g4x(gb[j & 1], qx, qx.tau_x, ptr, cd[4 * j], cd[4 * j + 1], cd[4 * j + 2],
                         cd[4 * j + 3]);
                if ((j & 3) == 3 && ptr > llim) {
                    overflow = true;
                    ptr = llim;
                }
            }
        } else {
            G4 gb[2];
            load_g4(gb[0], base, 0);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (j + 1 < 8) load_g4(gb[(j + 1) & 1], base, 4 * (j + 1));
                eval_g4(gb[j & 1], qv, tau, ptr, cd[4 * j], cd[4 * j + 1], cd[4 * j + 2], cd[4 * j + 3]);
                if ((j & 3) == 3 && ptr > llim) {  // clamp every 16 candidates (kSlack)
                    overflow = true;
                    ptr = llim;
                }
            }
        }
        __syncwarp();
        head ^= 32;
        filled = max(filled - 32, 0);
    }
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

// Finish query j of the tile (warp-cooperative; lanes over its list entries):
// float64 keys in the reference's operation order (pyx:32-48, no FMA) ->
// float32 keys; certificate (>= need entries strictly inside tau_j); counting
// sort into kBkt buckets on (key/tau)^(d/2) (uniform for uniform density) with
// __match_any groups; odd-even transposition inside buckets; equal float32
// keys among the decided entries -> exact path; the sorted row (self first) is
// written coalesced.  Returns false when the query must be redone.
constexpr int kRounds = (kCap + 31) / 32;
#ifndef FG_FINISH_MATCH
#define FG_FINISH_MATCH 0
#endif

// Global gathers of one query's list (coordinates and original ids of its
// entries): issued for query j+1 while query j is being finished.
struct QLoads {
    float4 c[kRounds];
    int32_t cpos[kRounds];
    int32_t id[kRounds];
    int m;
};

__device__ __forceinline__ void fetch_query(const ScanWarp& W, const TileArgs& a, int j, int m_l,
                                            QLoads& Q) {
    const int lane = lane_id();
    Q.m = __shfl_sync(FG_FULL_MASK, m_l, j);
    const uint16_t* L = &W.code[j * kStride];
#pragma unroll
    for (int t = 0; t < kRounds; ++t) {
        const int e = lane + 32 * t;
        Q.cpos[t] = -1;
        if (32 * t < Q.m && e < Q.m) {  // 32t < m is warp-uniform
            const uint16_t cd = L[e];
            Q.cpos[t] = W.spS[cd >> 7] + (cd & 127);
            Q.c[t] = a.sc[Q.cpos[t]];
            Q.id[t] = a.sid[Q.cpos[t]];
        }
    }
}

template <int DB, class WS>
__device__ __forceinline__ bool finish_query(WS& W, const TileArgs& a, int j, const QLoads& Q,
                                             const float4 q, int32_t p, float tau, int32_t qid_l,
                                             int need) {
    const float qa[4] = {q.x, q.y, q.z, q.w};
    const int lane = lane_id();
    const int m = Q.m;
    const int32_t pj = __shfl_sync(FG_FULL_MASK, p, j);
    const float tj = __shfl_sync(FG_FULL_MASK, tau, j);
    double qd[DB];
#pragma unroll
    for (int i = 0; i < DB; ++i) qd[i] = (double)__shfl_sync(FG_FULL_MASK, qa[i], j);
    const float inner = tj * (1.0f - 3e-5f);
    const float inv_tau = 1.0f / tj;
    constexpr int R = kRounds;
    float key[R];
#pragma unroll
    for (int t = 0; t < R; ++t) key[t] = kInf;
    const int32_t* cpos = Q.cpos;
    const float4* c = Q.c;
    int n_in = 0;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        if (cpos[t] >= 0 && cpos[t] != pj) {
            const float cc[4] = {c[t].x, c[t].y, c[t].z, c[t].w};
            double acc = 0.0;
#pragma unroll
            for (int i = 0; i < DB; ++i) {
                const double d = __dsub_rn(qd[i], (double)cc[i]);
                acc = i == 0 ? __dmul_rn(d, d) : __dadd_rn(acc, __dmul_rn(d, d));
            }
            key[t] = __double2float_rn(acc);
            n_in += key[t] < inner ? 1 : 0;
        }
    }
    if (__reduce_add_sync(FG_FULL_MASK, n_in) < need) return false;
    // counting sort by bucket: counts (match_any groups + one smem atomic per group)
    *reinterpret_cast<uint4*>(&W.bcnt[4 * lane]) = make_uint4(0u, 0u, 0u, 0u);
    __syncwarp();
    int bk[R], idx[R];
#pragma unroll
    for (int t = 0; t < R; ++t) {
        bk[t] = key[t] < kInf ? bucket_of<DB>(key[t], inv_tau) : kBkt;
        idx[t] = 0;
#if FG_FINISH_MATCH
        if (32 * t < m) {
            const unsigned mm = __match_any_sync(FG_FULL_MASK, bk[t]);
            const int leader = __ffs(mm) - 1;
            unsigned old = 0;
            if (lane == leader && bk[t] < kBkt)
                old = atomicAdd(&W.bcnt[bk[t]], (unsigned)__popc(mm));
            idx[t] = (int)__shfl_sync(FG_FULL_MASK, old, leader) + __popc(mm & lanemask_lt());
        }
#else
        // one shared-memory atomic per entry (native integer add; bucket mates
        // in one warp instruction serialise, rare at ~0.45 entries per bucket);
        // the in-bucket order this leaves is undone by the (key, position) rank
        if (bk[t] < kBkt) idx[t] = (int)atomicAdd(&W.bcnt[bk[t]], 1u);
#endif
    }
    __syncwarp();
    uint4 ca = *reinterpret_cast<const uint4*>(&W.bcnt[4 * lane]);
    const unsigned tot = ca.x + ca.y + ca.z + ca.w;
    const unsigned incl = warp_inclusive_scan(tot);
    const int n_valid = (int)__shfl_sync(FG_FULL_MASK, incl, 31);
    __syncwarp();
    {  // exclusive starts of this lane's 4 buckets
        unsigned run = incl - tot, t0;
        t0 = ca.x; ca.x = run; run += t0;
        t0 = ca.y; ca.y = run; run += t0;
        t0 = ca.z; ca.z = run; run += t0;
        ca.w = run;
    }
    *reinterpret_cast<uint4*>(&W.bcnt[4 * lane]) = ca;
    if (lane == 31) W.bcnt[kBkt] = incl;
    __syncwarp();
#pragma unroll
    for (int t = 0; t < R; ++t) {
        if (bk[t] < kBkt) {
            const int at = (int)W.bcnt[bk[t]] + idx[t];
            W.skey[at] = key[t];
            W.sid[at] = Q.id[t];
        }
    }
    __syncwarp();
    // final slot = bucket start + rank inside the bucket (a uniform maxb-step
    // loop); only buckets starting at or below `need` can reach the decided
    // range.  Equal float32 keys there: the exact path decides.
    bool amb = false;
#pragma unroll
    for (int t = 0; t < R; ++t) {
        const int sl = lane + 32 * t;
        if (32 * t < n_valid) {
            const bool valid = sl < n_valid;
            const float kk = W.skey[valid ? sl : 0];
            const int b = bucket_of<DB>(kk, inv_tau);
            const int b0 = (int)W.bcnt[b], b1 = (int)W.bcnt[b + 1];
            const bool live = valid && b0 <= need;
            int r = b0;
            bool tie = false;
            if (live) {
                if (b1 - b0 <= 3) {  // the common case: unrolled, no loop
                    // keys are >= 0: their bit patterns order like the floats, so
                    // (key, position) compares as one 64-bit integer
                    const unsigned kb = __float_as_uint(kk);
                    const unsigned long long me = ((unsigned long long)kb << 32) | (unsigned)sl;
#pragma unroll
                    for (int u = 0; u < 3; ++u) {
                        const int i = b0 + u;
                        const unsigned ib = __float_as_uint(W.skey[min(i, kCap - 1)]);
                        const unsigned long long other = ((unsigned long long)ib << 32) | (unsigned)i;
                        r += (i < b1 && other < me) ? 1 : 0;
                        tie |= i < b1 && i != sl && ib == kb;
                    }
                } else {
                    for (int i = b0; i < b1; ++i) {
                        const float ki = W.skey[i];
                        r += (ki < kk || (ki == kk && i < sl)) ? 1 : 0;
                        tie |= ki == kk && i != sl;
                    }
                }
            }
            if (live) {
                W.okey[r + 1] = kk;
                W.oid[r + 1] = W.sid[sl];
            }
            amb |= tie && r < need;
        }
    }
    if (__any_sync(FG_FULL_MASK, amb)) return false;
    const int32_t qid = __shfl_sync(FG_FULL_MASK, qid_l, j);
    if (lane == 0) {
        W.okey[0] = 0.0f;
        W.oid[0] = qid;
    }
    __syncwarp();
    int32_t* oi = a.out_idx + (int64_t)qid * a.k;
    float* od = a.out_d2 + (int64_t)qid * a.k;
    if ((a.k & 3) == 0) {  // 16-byte row segments
        for (int g = lane; 4 * g < a.k; g += 32) {
            *reinterpret_cast<int4*>(oi + 4 * g) = *reinterpret_cast<const int4*>(&W.oid[4 * g]);
            *reinterpret_cast<float4*>(od + 4 * g) = *reinterpret_cast<const float4*>(&W.okey[4 * g]);
        }
    } else {
        for (int sl = lane; sl < a.k; sl += 32) {
            oi[sl] = W.oid[sl];
            od[sl] = W.okey[sl];
        }
    }
    __syncwarp();
    return true;
}

// ---------------------------------------------------------------- search
template <int DB, bool SPLIT>
__global__ void __launch_bounds__(kWarps * 32, SPLIT ? kScanCtasPerSm : kCtasPerSm)
    k_tile_search(const __grid_constant__ TileArgs a) {
    constexpr int NL = DB - 1;
    using WT = typename std::conditional<SPLIT, ScanWarp, TileWarp>::type;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WT& W = reinterpret_cast<WT*>(smem_raw)[threadIdx.x >> 5];
    const int lane = lane_id();
    const int nb = a.nb;
    const int need = a.k - 1;
    const int n_tiles = tiles_declined(a) ? 0 : a.ctr[0];
    if (a.hint && blockIdx.x == 0 && threadIdx.x == 0) *a.hint = tiles_declined(a) ? 1 : 0;
    unsigned long long st_cand = 0, st_tiles = 0, st_redo = 0, st_fail = 0, st_exp = 0, st_eval = 0;

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
                    if (a.meta && i0 + lane < L) a.meta[S + i0 + lane] = make_float2(0.f, -1.f);
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
        // only lanes within reach of a face of the grid box need the correction
        // (a radius <= 3 r_k: the ball of the first iteration can grow by f^(-1/d))
        bool near_face = false;
#pragma unroll
        for (int i = 0; i < DB; ++i) {
            const float h0 = qa[i] - mn[i];
            near_face |= fminf(h0, (float)nb * w[i] - h0) < 3.0f * rad;
        }
#pragma unroll 1
        for (int it = 0; it < (__any_sync(FG_FULL_MASK, active && near_face) ? FG_RADIUS_ITERS : 0); ++it) {
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
            if (a.meta && active) a.meta[p] = make_float2(0.f, -1.f);
            st_redo += active ? 1 : 0;
            __syncwarp();
            continue;
        }
        if (lane == 0) W.spE[nsp] = (uint16_t)T;
        __syncwarp();
        st_cand += T;

        // ---- scan: 32 candidates per chunk, broadcast to every lane
        const QP qv = pack_q(q);
        const uint32_t lbase = (uint32_t)__cvta_generic_to_shared(&W.code[lane * kStride]);
        const uint32_t llim = lbase + kCap * 2;
        uint32_t ptr = lbase;
        bool overflow = false;
        // expanded form around the bbox centre when its error bound allows
        float cq[4] = {0.f, 0.f, 0.f, 0.f};
        float rc2 = 0.0f;
#pragma unroll
        for (int i = 0; i < DB; ++i) {
            cq[i] = mn[i] + 0.5f * (lo[i] + hi[i]) * w[i];
            const float rci = rr_max * invw[i] + kSlackCells;
            const float blo = mn[i] + fmaxf(floorf(lo[i] - rci), 0.0f) * w[i];
            const float bhi = mn[i] + (fminf(floorf(hi[i] + rci), (float)(nb - 1)) + 1.0f) * w[i];
            const float e = fmaxf(fabsf(blo - cq[i]), fabsf(bhi - cq[i]));
            rc2 = fmaf(e, e, rc2);
        }
        const float4 cen = make_float4(cq[0], cq[1], cq[2], cq[3]);
        const float4 qs = make_float4(q.x - cen.x, q.y - cen.y, q.z - cen.z, q.w - cen.w);
        const float sq = fmaf(qs.w, qs.w, fmaf(qs.z, qs.z, fmaf(qs.y, qs.y, qs.x * qs.x)));
        const float rq = warp_max_f(active ? sqrtf(sq) : 0.0f);
        const float tau_min = warp_min_f(active ? tau : kInf);
        const float rsum = (rq + sqrtf(rc2)) * 1.01f;
#ifndef FG_TILE_EXPANDED
#define FG_TILE_EXPANDED 0
#endif
        const bool expanded = FG_TILE_EXPANDED && rsum * rsum <= 32.0f * tau_min;
        QX qx;
        qx.sq = pack2(sq);
        qx.m2q[0] = pack2(-2.0f * qs.x);
        qx.m2q[1] = pack2(-2.0f * qs.y);
        qx.m2q[2] = pack2(-2.0f * qs.z);
        qx.m2q[3] = pack2(-2.0f * qs.w);
        qx.tau_x = tau - sq;
        st_exp += expanded ? 1 : 0;
        {
            float bl[4] = {0.f, 0.f, 0.f, 0.f}, bh[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int i = 0; i < DB; ++i) {  // the queries' physical bounding box
                bl[i] = warp_min_f(active ? qa[i] : kInf);
                bh[i] = warp_max_f(active ? qa[i] : -kInf);
            }
            const float thr = tau_max * kMargin + 1e-30f;
            if (expanded)
                scan_tile_filtered<true>(W, a.sc, T, nsp, qv, qx, cen, tau,
                                         make_float4(bl[0], bl[1], bl[2], bl[3]),
                                         make_float4(bh[0], bh[1], bh[2], bh[3]), thr, ptr, overflow,
                                         llim, st_eval);
            else
            scan_tile_filtered<false>(W, a.sc, T, nsp, qv, qx, cen, tau, make_float4(bl[0], bl[1], bl[2], bl[3]),
                               make_float4(bh[0], bh[1], bh[2], bh[3]), thr, ptr, overflow, llim,
                               st_eval);
        }
        asm volatile("" ::: "memory");  // list stores (inline asm) before the epilogue reads

        // ---- epilogue: the warp finishes the lanes' queries one at a time
        const int m_l = (int)(ptr - lbase) >> 1;
#if defined(FG_TILE_SCAN_ONLY)  // timing experiment: no epilogue (wrong results)
        if (active && m_l == 1000) a.out_idx[p] = m_l;
        __syncwarp();
        continue;
#endif
        if constexpr (SPLIT) {  // split epilogue: hand the lists to k_tile_finish
            if (active && !overflow) {
                const uint16_t* L = &W.code[lane * kStride];
                int4* dst = reinterpret_cast<int4*>(a.lists + (int64_t)p * kCap);
                for (int e = 0; e < m_l; e += 4) {
                    int32_t v4[4];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint16_t cd = L[min(e + u, m_l - 1)];
                        v4[u] = W.spS[cd >> 7] + (cd & 127);
                    }
                    dst[e >> 2] = make_int4(v4[0], v4[1], v4[2], v4[3]);
                }
                a.meta[p] = make_float2(tau, (float)m_l);
            }
            const bool redo = active && overflow;
            if (redo) a.meta[p] = make_float2(0.f, -1.f);
            push_redo(a, redo, p);
            st_redo += redo ? 1 : 0;
            __syncwarp();
            continue;
        }
        if constexpr (!SPLIT) {
            const unsigned todo = __ballot_sync(FG_FULL_MASK, active && !overflow);
            bool ok = false;  // this lane's query got its row
            const int32_t qid_l = active ? a.sid[p] : 0;
            QLoads cur, nxt;
            if (todo) fetch_query(W, a, __ffs(todo) - 1, m_l, cur);
            for (unsigned mask = todo; mask;) {
                const int j = __ffs(mask) - 1;
                mask &= mask - 1;
                if (mask) fetch_query(W, a, __ffs(mask) - 1, m_l, nxt);  // next query's gathers
                const bool okj = finish_query<DB>(W, a, j, cur, q, p, tau, qid_l, need);
                if (lane == j) ok = okj;
                cur = nxt;
            }
            const bool redo = active && !ok;
            push_redo(a, redo, p);
            st_redo += redo ? 1 : 0;
            __syncwarp();
        }
    }
    if (a.stats) {
        st_redo = __reduce_add_sync(FG_FULL_MASK, (unsigned)st_redo);
        if (lane == 0) {
            atomicAdd(&a.stats[TS_TILES], st_tiles);
            atomicAdd(&a.stats[TS_CAND], st_cand);
            atomicAdd(&a.stats[TS_REDO], st_redo);
            atomicAdd(&a.stats[TS_TILE_FAIL], st_fail);
            atomicAdd(&a.stats[TS_EXPANDED], st_exp);
            atomicAdd(&a.stats[TS_EVAL], st_eval);
        }
    }
}

// ---------------------------------------------------------------- split epilogue
struct FinishWarp {
    float skey[kCap];
    int32_t sid[kCap];
    alignas(16) float okey[kCap + 4];
    alignas(16) int32_t oid[kCap + 4];
    alignas(16) uint32_t bcnt[kBkt + 4];
};
constexpr int kFinishWarps = 8;
#ifndef FG_FINISH_MINB
#define FG_FINISH_MINB 4
#endif

// Warp per query in sorted order (neighbouring warps share candidates in L1/L2),
// the lists written by k_tile_search; the same finish_query as the fused path.
template <int DB>
__global__ void __launch_bounds__(kFinishWarps * 32, FG_FINISH_MINB) k_tile_finish(const __grid_constant__ TileArgs a,
                                                                   int64_t n) {
    __shared__ FinishWarp fw[kFinishWarps];
    FinishWarp& W = fw[threadIdx.x >> 5];
    const int lane = lane_id();
    const int need = a.k - 1;
    unsigned long long st_redo = 0;
    if (tiles_declined(a)) return;
#ifndef FG_FINISH_PREFETCH
#define FG_FINISH_PREFETCH 1
#endif
#if FG_FINISH_PREFETCH
    // the next query's meta and list entries are loaded while this one is
    // finished (the list row is read whole, without waiting for its length):
    // only the coordinate / id gathers stay on the per-query critical path
    // two-deep: the meta of query p + 2 stride and the list entries of query
    // p + stride (only its m of them: the meta arrived an iteration earlier)
    // load while query p is finished
    const int64_t stride = (int64_t)gridDim.x * kFinishWarps;
    int64_t p = blockIdx.x * (int64_t)kFinishWarps + (threadIdx.x >> 5);
    float2 mt = p < n ? a.meta[p] : make_float2(0.f, -1.f);
    float2 mt_n = p + stride < n ? a.meta[p + stride] : make_float2(0.f, -1.f);
    int32_t lnext[kRounds];
#pragma unroll
    for (int t = 0; t < kRounds; ++t)
        lnext[t] = lane + 32 * t < (int)mt.y ? a.lists[p * kCap + lane + 32 * t] : -1;
    for (; p < n; p += stride) {
        const int m = (int)mt.y;
        const float tau_p = mt.x;
        QLoads Q;
        Q.m = m;
#pragma unroll
        for (int t = 0; t < kRounds; ++t) Q.cpos[t] = lnext[t];
        const int64_t pn = p + stride, pnn = p + 2 * stride;
        const int mn = (int)mt_n.y;
#pragma unroll
        for (int t = 0; t < kRounds; ++t)
            lnext[t] = lane + 32 * t < mn ? a.lists[pn * kCap + lane + 32 * t] : -1;
        mt = mt_n;
        mt_n = pnn < n ? a.meta[pnn] : make_float2(0.f, -1.f);
        if (m < 0) continue;  // already on the redo list
#pragma unroll
        for (int t = 0; t < kRounds; ++t) {
            const int e = lane + 32 * t;
            if (32 * t < m && e < m) {
                Q.c[t] = a.sc[Q.cpos[t]];
                Q.id[t] = a.sid[Q.cpos[t]];
            } else {
                Q.cpos[t] = -1;
            }
        }
        const float4 q = a.sc[p];
        const int32_t qid = a.sid[p];
        const bool ok = finish_query<DB>(W, a, 0, Q, q, (int32_t)p, tau_p, qid, need);
        if (!ok && lane == 0) {
            a.redo[atomicAdd(&a.ctr[2], 1)] = (int32_t)p;
            ++st_redo;
        }
        __syncwarp();
    }
#else
    for (int64_t p = blockIdx.x * (int64_t)kFinishWarps + (threadIdx.x >> 5); p < n;
         p += (int64_t)gridDim.x * kFinishWarps) {
        const float2 mt = a.meta[p];
        const int m = (int)mt.y;
        if (m < 0) continue;  // already on the redo list
        QLoads Q;
        Q.m = m;
        const int32_t* lp = a.lists + p * kCap;
#pragma unroll
        for (int t = 0; t < kRounds; ++t) {
            const int e = lane + 32 * t;
            Q.cpos[t] = -1;
            if (32 * t < m && e < m) {
                Q.cpos[t] = lp[e];
                Q.c[t] = a.sc[Q.cpos[t]];
                Q.id[t] = a.sid[Q.cpos[t]];
            }
        }
        const float4 q = a.sc[p];
        const int32_t qid = a.sid[p];
        const bool ok = finish_query<DB>(W, a, 0, Q, q, (int32_t)p, mt.x, qid, need);
        if (!ok && lane == 0) {
            a.redo[atomicAdd(&a.ctr[2], 1)] = (int32_t)p;
            ++st_redo;
        }
        __syncwarp();
    }
#endif
    if (a.stats && lane == 0 && st_redo) atomicAdd(&a.stats[TS_REDO], st_redo);
}

}  // namespace tile
}  // namespace fg
