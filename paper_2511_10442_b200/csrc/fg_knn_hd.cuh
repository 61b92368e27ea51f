// fg_knn_hd.cuh -- binned_select_knn forward, lane-per-query tiles for the
// cases the d <= 4 tile path does not take: more than 4 coordinates, or fewer
// binned dims than coordinates (config C: 1M x 10, d_bin 5, k 64).  Replaces
// pyx:188-329 for those shapes; same canonical answer.
//
// The warp-per-query kernel spends ~90 warp instructions per 32 candidates of
// one query on region bookkeeping; at d = 10 a query scans ~10^5 candidates.
// Here one warp owns a tile of 32 spatially compact queries (lane = query) and
// every candidate is loaded once into shared memory and evaluated by all 32
// lanes with packed fp32x2 arithmetic (FADD2 + FFMA2 over candidate pairs):
// ~DE/2 + 1 warp instructions per candidate for 32 (query, candidate) pairs.
//
// * tiles (k_hd_tiles): the block of 2^(DB-1) lead rows x all last-dim cells
//   (tile path blocks) is cut into runs of exactly 32 points in column-major
//   (last-dim cell, lead row) order -- compact boxes, full warps.
// * per tile: lane buffers of (fp32 d2, sorted position) in shared memory
//   (kCap entries); a candidate enters lane l's buffer iff its fp32 d2 <=
//   tau_l.  A full buffer (checked per group of 4 candidates) is cut by a
//   warp-cooperative radix select to the (need+1) smallest (self included) and
//   tau_l drops to that value x (1+1e-5).
// * region growth: stage radius rho; the region is every lead row whose box
//   distance (binned dims) to the tile's query box is <= rho, trimmed along the
//   last binned dim; stage i scans only the shell between the regions of rho_{i-1}
//   and rho_i (recomputed with identical float operations, so no cell is scanned
//   twice or skipped).  After a stage every lane's tau_l is tightened to its
//   (need+1)-th smallest entry; the search stops when sqrt(max_l tau_l) <= rho:
//   the binned distance never exceeds the full distance, so the region holds
//   every point within each lane's tau_l.  rho_1 comes from the previous tile
//   of the same warp (neighbouring tiles, similar radii).
// * epilogue: lane j's buffer (self dropped) is handed to the warp-per-query
//   kernel's exact epilogue (float64 keys in the reference's operation order,
//   pyx:32-48; (d2_f64, index) order) one lane at a time.
// * a buffer the radix cut cannot shrink (> kCap - 8 entries within 1e-5 of
//   each other: duplicates) keeps exactly the need+1 smallest by (float64 key,
//   index) instead -- no fallback kernel.
// * float64 coordinates (fg_knn_fwd_f64_ws): exact keys from the float64 values;
//   the fp32 filter compares against (sqrt(x) + r)^2, r bounding the float32
//   rounding of coordinate differences (k_abs_bound), so no true neighbour is
//   filtered out.
#pragma once

#include "fg_knn_tile.cuh"

namespace fg {
namespace hd {

#ifndef FG_HD_WARPS
#define FG_HD_WARPS 2
#endif
constexpr int kWarps = FG_HD_WARPS;  // warps per CTA
#ifndef FG_HD_UNROLL
#define FG_HD_UNROLL 4
#endif
constexpr int kUnroll = FG_HD_UNROLL;  // 4-candidate groups in flight per chunk
#ifndef FG_HD_HINT_SCALE
#define FG_HD_HINT_SCALE 0.5f
#endif
constexpr float kHintScale = FG_HD_HINT_SCALE;  // first-stage radius^2 / previous tile's
#ifndef FG_HD_SEED
#define FG_HD_SEED 120
#endif
constexpr int kSeed = FG_HD_SEED;  // stage-0 tau seeding window (sorted positions), 0: off
static_assert(kSeed < 256, "8-bit seed bucket counters");
#ifndef FG_HD_CAP
#define FG_HD_CAP 128
#endif
constexpr int kCap = FG_HD_CAP;  // per-lane buffer entries
#ifndef FG_HD_FILTER_DE
#define FG_HD_FILTER_DE 4
#endif
// candidates are filtered against the tile's query box for DE <= this (the
// clustered d <= 4 fallback: dense cells are scanned whole at cell granularity)
constexpr int kFilterDE = FG_HD_FILTER_DE;
constexpr int kMaxNeed1 = 64;  // host eligibility (float32 coordinates): k <= 64
constexpr int kMaxK64 = kCap - 8;  // float64 coordinates: k <= 120 (a cut frees >= 4 slots)
constexpr float kMargin = 1.0f + 1e-5f;
constexpr float kTiny = 1e-35f;
constexpr float kSlackCells = 1e-4f;
constexpr float kInf = __builtin_huge_valf();

enum { HS_TILES, HS_CHUNKS, HS_STAGES, HS_MAXCYC, HS_COMPACT, HS_COUNT };  // HS_MAXCYC: slowest tile (clock64)

template <int DE, int CAP>
struct HdWarp {
    static constexpr int kStride = CAP + 1;
    float bd[32 * kStride];    // lane buffers: fp32 d2 (odd stride: appends spread over banks)
    int32_t bp[32 * kStride];  //               sorted positions
    // candidates, SoA: a 64-entry ring when filtered, else one 32-candidate
    // chunk (at DE = 10 the extra 2.6 KB per warp would cost a CTA per SM)
    alignas(16) float sx[DE][DE <= kFilterDE ? 64 : 32];
    alignas(16) int32_t spos[DE <= kFilterDE ? 64 : 32];
    int32_t span_s[64], span_l[64];
    search::WarpBuf<128> eb;   // epilogue scratch (the warp-per-query kernel's)
};

// Per-lane buffer entries and warps per CTA of an instantiation: the float32
// d <= 4 kernels (the clustered fallback, k <= 41 there) use 80 entries and
// one warp per CTA -- 9 warps/SM (the 224-register cap allows 9) instead of 6
// with 128 (config B: 96 entries / 7 warps 8% faster than 128, 80 / 9 warps
// another ~10%; 72 entries at 200 registers / 10 warps no faster, 64 entries
// at 168 registers spill); d > 4 (config C, k = 64: more room between cuts)
// and float64 (k <= 120) keep 128.
#ifndef FG_HD_CAP_LOWD
#define FG_HD_CAP_LOWD 80
#endif
template <int NV, bool X64>
__host__ __device__ constexpr int hd_cap() {
    return NV == 1 && !X64 ? FG_HD_CAP_LOWD : kCap;
}
template <int NV, bool X64>
__host__ __device__ constexpr int hd_warps() {
    return NV == 1 && !X64 ? 1 : kWarps;
}
template <int DE, int CAP, int WARPS>
__host__ __device__ constexpr size_t hd_smem_bytes() {
    return sizeof(HdWarp<DE, CAP>) * WARPS;
}

// ---------------------------------------------------------------- tile list
// One warp per (split, lead block): lane c owns last-dim column c (nb <= 32);
// the block's points in (column, row) order are cut into runs of <= 32 that
// never span more than kTileSpan columns: in a sparse block 32 consecutive
// points can lie in columns far apart, and a tile's region is the union of
// its queries' -- one elongated tile then scans most of the split (config B:
// a single such tile took 2 ms).
constexpr int kTileSpan = 2;

template <int DB>
__global__ void __launch_bounds__(128) k_hd_tiles(const tile::TileArgs a) {
    constexpr int NL = DB - 1;
    const int lane = lane_id();
    const int blk = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (blk >= a.n_blocks || tile::gated_off(a)) return;
    const int s = blk / a.bps;
    int o[NL > 0 ? NL : 1];
    tile::block_origin<NL>(blk - s * a.bps, a.nblk, o);
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
    // the cut (warp-uniform walk over the columns): pass 0 counts, pass 1 writes
    int t0 = 0;
    for (int pass = 0; pass < 2; ++pass) {
        int nt = 0, run = 0, c0 = 0, g0 = 0, g = 0;
        auto emit = [&](int start, int len) {
            if (pass == 1 && lane == 0) {
                a.tiles[t0 + nt] = make_int2(blk, start);
                a.tcnt[t0 + nt] = (uint8_t)len;
            }
            ++nt;
        };
        for (int c = 0; c < nb; ++c) {
            int cnt = __shfl_sync(FG_FULL_MASK, col, c);
            if (cnt == 0) continue;
            if (run > 0 && c - c0 >= kTileSpan) {
                emit(g0, run);
                run = 0;
            }
            if (run > 0) {  // top up the open run
                const int take = min(cnt, 32 - run);
                run += take;
                cnt -= take;
                g += take;
                if (run == 32) {
                    emit(g0, run);
                    run = 0;
                }
            }
            if (cnt >= 32) {  // whole runs of this column, written in parallel
                const int nf = cnt >> 5;
                if (pass == 1)
                    for (int i = lane; i < nf; i += 32) {
                        a.tiles[t0 + nt + i] = make_int2(blk, g + 32 * i);
                        a.tcnt[t0 + nt + i] = (uint8_t)32;
                    }
                nt += nf;
                g += 32 * nf;
                cnt -= 32 * nf;
            }
            if (cnt > 0) {  // a new open run
                c0 = c;
                g0 = g;
                run = cnt;
                g += cnt;
            }
        }
        if (run > 0) emit(g0, run);
        if (pass == 0) {
            if (lane == 0 && nt > 0) t0 = atomicAdd(&a.ctr[0], nt);
            t0 = __shfl_sync(FG_FULL_MASK, t0, 0);
        }
    }
}

// Lane -> sorted position of tile ti's point `lane` (-1: none): the block's
// points in (column, row) order, lanes [0, tcnt) from the tile's start.
template <int DB>
__device__ __forceinline__ int32_t tile_point(const tile::TileArgs& t, int ti) {
    constexpr int NL = DB - 1;
    const int lane = lane_id();
    const int2 td = t.tiles[ti];
    const int blk = td.x, start = td.y, tlen = t.tcnt[ti];
    const int s = blk / t.bps;
    int o[NL > 0 ? NL : 1];
    tile::block_origin<NL>(blk - s * t.bps, t.nblk, o);
    const int64_t cbase = (int64_t)s * t.total;
    const int nb = t.nb;
    int col = 0;
    if (lane < nb) {
#pragma unroll
        for (int rr = 0; rr < (1 << NL); ++rr) {
            int rowflat = 0;
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int j = o[i] + ((rr >> (NL - 1 - i)) & 1);
                ok &= j < nb;
                rowflat = rowflat * nb + j;
            }
            if (ok) {
                const int64_t rc = cbase + (int64_t)rowflat * nb + lane;
                col += t.bounds[rc + 1] - t.bounds[rc];
            }
        }
    }
    const int P = warp_inclusive_scan(col);
    const int g = start + lane;
    int c = 0;
    for (int cc = 0; cc < nb; ++cc) c += __shfl_sync(FG_FULL_MASK, P, cc) <= g ? 1 : 0;
    const int Ptot = __shfl_sync(FG_FULL_MASK, P, 31);
    const int Pprev = __shfl_sync(FG_FULL_MASK, P, max(c - 1, 0));
    int32_t p = -1;
    if (lane < tlen && g < Ptot && c < nb) {
        int off = g - (c > 0 ? Pprev : 0);
        for (int rr = 0; rr < (1 << NL); ++rr) {
            int rowflat = 0;
            bool ok = true;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                const int j = o[i] + ((rr >> (NL - 1 - i)) & 1);
                ok &= j < nb;
                rowflat = rowflat * nb + j;
            }
            if (!ok) continue;
            const int64_t rc = cbase + (int64_t)rowflat * nb + c;
            const int32_t b0 = t.bounds[rc], len = t.bounds[rc + 1] - b0;
            if (off < len) {
                p = b0 + off;
                break;
            }
            off -= len;
        }
    }
    return p;
}

// Dispatch order: a tile's cost grows with its query box (a wide box reaches
// far more candidates), and a costly tile taken last is the kernel's tail
// (config B: one tile took half the kernel's time).  Tiles are counted into
// 64 buckets of log2(box diagonal^2) (k_hd_cost), the buckets laid out widest
// first (k_hd_rank) and the tiles placed (k_hd_place); the search takes them in
// that order.
constexpr int kCostBuckets = 64;

template <int NV, int DB>
__global__ void __launch_bounds__(128) k_hd_cost(const tile::TileArgs t) {
    const int ti = blockIdx.x * 4 + (threadIdx.x >> 5);
    if (ti >= t.ctr[0] || tile::gated_off(t)) return;
    const int32_t p = tile_point<DB>(t, ti);
    const bool live = p >= 0;
    const float4 x = live ? t.sc[(int64_t)p * NV] : make_float4(0.f, 0.f, 0.f, 0.f);
    float d2 = 0.0f;
    const float xa[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int d = 0; d < 4; ++d) {
        const float e = tile::warp_max_f(live ? xa[d] : -kInf) - tile::warp_min_f(live ? xa[d] : kInf);
        d2 = fmaf(e, e, d2);
    }
    if (lane_id() == 0) {
        int b = 0;  // bucket 0: the widest boxes
        if (d2 > 0.0f && d2 < kInf) b = min(max(40 - ilogbf(d2), 0), kCostBuckets - 1);
        if (!(d2 < kInf)) b = 0;
        t.tkey[ti] = (uint8_t)b;
        atomicAdd(&t.hist[b], 1);
    }
}

static __global__ void k_hd_rank(const tile::TileArgs t) {
    if (tile::gated_off(t)) return;
    const int lane = threadIdx.x;  // one warp: 64 buckets, 2 per lane
    const int a0 = t.hist[2 * lane], a1 = t.hist[2 * lane + 1];
    const int incl = warp_inclusive_scan(a0 + a1);
    t.hist[kCostBuckets + 2 * lane] = incl - a0 - a1;
    t.hist[kCostBuckets + 2 * lane + 1] = incl - a1;
}

static __global__ void __launch_bounds__(256) k_hd_place(const tile::TileArgs t) {
    const int ti = blockIdx.x * blockDim.x + threadIdx.x;
    if (ti >= t.ctr[0] || tile::gated_off(t)) return;
    t.order[atomicAdd(&t.hist[kCostBuckets + t.tkey[ti]], 1)] = ti;
}

// ---------------------------------------------------------------- helpers
__device__ __forceinline__ unsigned long long dup2(float x) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
    return r;
}

// Region geometry of one stage: lead-dim enumeration box and the radius.
template <int NL>
struct Box {
    int L[NL > 0 ? NL : 1], N[NL > 0 ? NL : 1];
    float inv[NL > 0 ? NL : 1];
    int rows;
    float rho2;   // radius^2 (physical units); < 0: empty region
    float slack;  // cell units
};

template <int DB>
__device__ __forceinline__ Box<DB - 1> make_box(float rho2, const float (&lo)[DB], const float (&hi)[DB],
                                               const float (&invw)[DB], int nb, float slack) {
    constexpr int NL = DB - 1;
    Box<NL> b;
    b.rho2 = rho2;
    b.slack = slack;
    b.rows = rho2 < 0.0f ? 0 : 1;
    const float rho = sqrtf(fmaxf(rho2, 0.0f)) * kMargin;
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        const float rc = rho * invw[i] + slack;
        b.L[i] = (int)fmaxf(floorf(lo[i] - rc), 0.0f);
        b.N[i] = max((int)fminf(floorf(hi[i] + rc), (float)(nb - 1)) - b.L[i] + 1, 0);
        b.inv[i] = __frcp_rn((float)max(b.N[i], 1));
        b.rows *= b.N[i];
    }
    return b;
}

// Last-dim cell piece [ca, cb] of lead row jd inside the stage's region
// (ca > cb: empty).  Identical float operations for every caller.
template <int DB>
__device__ __forceinline__ void row_piece(const Box<DB - 1>& b, const int (&jd)[DB > 1 ? DB - 1 : 1],
                                          const float (&lo)[DB], const float (&hi)[DB],
                                          const float (&w)[DB], const float (&invw)[DB], int nb,
                                          int& ca, int& cb) {
    constexpr int NL = DB - 1;
    ca = 1;
    cb = 0;
    if (b.rho2 < 0.0f) return;
    bool inside = true;
    float bd2 = 0.0f;
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        inside &= jd[i] >= b.L[i] && jd[i] < b.L[i] + b.N[i];
        const float fj = (float)jd[i];
        float g = fmaxf(fmaxf(fj - hi[i], lo[i] - (fj + 1.0f)) - b.slack, 0.0f) * w[i];
        bd2 = fmaf(g, g, bd2);
    }
    const float rem = b.rho2 * (kMargin * kMargin) - bd2;
    if (!inside || rem < 0.0f) return;
    const float rc = sqrtf(rem) * invw[NL] * kMargin + b.slack;
    ca = (int)fmaxf(floorf(lo[NL] - rc), 0.0f);
    cb = (int)fminf(floorf(hi[NL] + rc), (float)(nb - 1));
}

// Exact float64 key of candidate cpos for the query (lane j's): the
// reference's operation order (pyx:32-48) on the float64 coordinates in
// float64 mode, on the float32 coordinates otherwise.
template <int NV, bool X64>
__device__ __forceinline__ double hd_key(const search::KnnArgs& a, const float (&qj)[4 * NV],
                                         int32_t qid, int32_t cpos) {
    if constexpr (X64) {
        const double* x = a.x64 + (int64_t)qid * a.n_c;
        const double* y = a.x64 + (int64_t)a.sid[cpos] * a.n_c;
        double acc = 0.0;
        for (int i = 0; i < a.n_c; ++i) {
            const double t = __dsub_rn(x[i], y[i]);
            acc = i == 0 ? __dmul_rn(t, t) : __dadd_rn(acc, __dmul_rn(t, t));
        }
        return acc;
    } else {
        float c[4 * NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 x = a.sc[(int64_t)cpos * NV + v];
            c[4 * v] = x.x; c[4 * v + 1] = x.y; c[4 * v + 2] = x.z; c[4 * v + 3] = x.w;
        }
        return exact_d2<4 * NV>(qj, c, a.n_c);
    }
}

// W.eb.p[0..m) -> (key, id, cp) with exact keys, sorted by (key, id); entries
// beyond max_radius2 get the sentinel.  Returns the sorted length (pow2).
template <int NV, bool X64, int DE, int CAP>
__device__ __noinline__ int exact_sort(HdWarp<DE, CAP>& W, const search::KnnArgs& a, int m,
                                       const float (&qj)[4 * NV], int32_t qid) {
    const int lane = lane_id();
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    int len = 32;
    while (len < m) len <<= 1;
    for (int e = lane; e < len; e += 32) {
        unsigned long long key = ~0ull;
        int32_t id = 0x7fffffff, cp = -1;
        if (e < m) {
            cp = W.eb.p[e];
            const double d = hd_key<NV, X64>(a, qj, qid, cp);
            if (!use_r2 || d <= a.max_r2) {
                key = (unsigned long long)__double_as_longlong(d);
                id = a.sid[cp];
            }
        }
        W.eb.key[e] = key;
        W.eb.id[e] = id;
        W.eb.cp[e] = cp;
    }
    __syncwarp();
    search::warp_sort_exact<128>(W.eb, len);
    return len;
}

// fp32 filter bound of a true squared distance x in float64 mode: a candidate
// whose float64 d2 is <= x has fp32 d2 (float32-rounded coordinates) <=
// (sqrt(x) + r)^2, r = sqrt(n_c) x max |coordinate difference error|.
__device__ __forceinline__ float up_bound(float x, float r) {
    const float s = sqrtf(x) + r;
    return s * s * kMargin + kTiny;
}

// Warp-cooperative cut of lane j's buffer to its keep smallest entries: P = an
// upper bound of the keep-th smallest fp32 d2 (16-bit radix select); the true bound tt_j
// becomes P (float64 mode: its upper bound) x (1+1e-5) and the filter
// threshold tau_j follows; entries above tau_j are dropped.  When near-ties
// leave no room (> kCap - 8 entries within the margin: duplicates), exactly
// the keep smallest by (float64 key, index) are kept -- the canonical order.
template <int NV, bool X64, int DE, int CAP>
__device__ __noinline__ int cut_lane(HdWarp<DE, CAP>& W, const search::KnnArgs& a, int j, int m, int keep,
                                     float& tau_j, float& tt_j, const float (&qj)[4 * NV],
                                     int32_t qid, float r) {
    const int lane = lane_id();
    constexpr int PER = (CAP + 31) / 32;  // CAP need not be a multiple of 32
    float* bd = &W.bd[j * (CAP + 1)];
    int32_t* bp = &W.bp[j * (CAP + 1)];
    __syncwarp();  // lane j's appends (its own shared-memory stores) before the other lanes read them
    unsigned key[PER];
    int32_t pv[PER];
    unsigned lo_k = 0xffffffffu, hi_k = 0u;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = i * 32 + lane;
        key[i] = e < m ? __float_as_uint(bd[e]) : 0xffffffffu;  // d2 >= 0: bits order like values
        pv[i] = e < m ? bp[e] : 0;
        if (e < m) {
            lo_k = min(lo_k, key[i]);
            hi_k = max(hi_k, key[i]);
        }
    }
    lo_k = __reduce_min_sync(FG_FULL_MASK, lo_k);
    hi_k = __reduce_max_sync(FG_FULL_MASK, hi_k);
    const float tt0 = __shfl_sync(FG_FULL_MASK, tt_j, j);
    // radix select on the top 16 bits (sign, exponent, 7 mantissa bits): P = an
    // upper bound of the keep-th smallest fp32 d2 within 2^-7 of it (the entries
    // sharing its 16-bit prefix stay; at most 16 rounds per cut).  A 32-bucket
    // histogram pass instead was measured no faster (C 262.7 vs 258.4 ms).
    const unsigned lo_p = lo_k >> 16, hi_p = hi_k >> 16;
    const int nbits = 32 - __clz(lo_p ^ hi_p);
    unsigned P = nbits >= 32 ? 0u : (lo_p & ~((1u << nbits) - 1u));
#pragma unroll 1
    for (int bit = nbits - 1; bit >= 0; --bit) {
        const unsigned t = P | ((1u << bit) - 1u);
        int c = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) c += (i * 32 + lane) < m && (key[i] >> 16) <= t ? 1 : 0;
        c = __reduce_add_sync(FG_FULL_MASK, c);
        if (c < keep) P |= 1u << bit;
    }
    const float Pf = __uint_as_float((P << 16) | 0xffffu);
    float tt = fminf(tt0, X64 ? up_bound(Pf, r) : Pf * kMargin + kTiny);
    float nt = X64 ? up_bound(tt, r) : tt;
    int kept = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i)
        kept += __popc(__ballot_sync(FG_FULL_MASK, (i * 32 + lane) < m && __uint_as_float(key[i]) <= nt));
    __syncwarp();
    int wpos = 0;
    if (kept <= CAP - 8) {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const bool k = (i * 32 + lane) < m && __uint_as_float(key[i]) <= nt;
            const unsigned bal = __ballot_sync(FG_FULL_MASK, k);
            if (k) {
                const int pos = wpos + __popc(bal & lanemask_lt());
                bd[pos] = __uint_as_float(key[i]);
                bp[pos] = pv[i];
            }
            wpos += __popc(bal);
        }
    } else {  // near-ties: the keep smallest by (float64 key, index)
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if (i * 32 + lane < m) W.eb.p[i * 32 + lane] = pv[i];
        __syncwarp();
        exact_sort<NV, X64, DE>(W, a, m, qj, qid);
        for (int e = lane; e < keep; e += 32) {  // valid keys sort first: a prefix
            const unsigned long long kk = W.eb.key[e];
            if (kk != ~0ull) {
                bd[e] = __double2float_ru(__longlong_as_double((long long)kk));
                bp[e] = W.eb.cp[e];
            }
        }
        __syncwarp();
        for (int e0 = 0; e0 < keep; e0 += 32)
            wpos += __popc(__ballot_sync(FG_FULL_MASK, e0 + lane < keep && W.eb.key[e0 + lane] != ~0ull));
        if (wpos >= keep) {
            const float f = __double2float_ru(__longlong_as_double((long long)W.eb.key[keep - 1]));
            tt = fminf(tt, f * kMargin + kTiny);
            nt = X64 ? up_bound(tt, r) : tt;
        }
    }
    __syncwarp();
    if (lane == j) {
        tau_j = nt;
        tt_j = tt;
    }
    return wpos;
}

// Stage-0 seed bound without buffers: every lane forms the fp32 d2 of the n
// sorted positions from w0 (n <= 255, real points of the split) and counts
// them in 32 quarter-octave buckets of x = d2 * s16 (8-bit counters packed in
// four registers; bucket 0: x < 1, bucket 31: unbounded).  Returns an upper
// bound of the lane's keep-th smallest d2 among them (the upper edge of the
// bucket where the count reaches keep; the largest d2 if only the open bucket
// does; +inf with fewer than keep points) -- within 25% of the value.
template <int NV, int DE, int CAP>
__device__ __forceinline__ float seed_bound(HdWarp<DE, CAP>& W, const search::KnnArgs& a, int64_t w0, int n,
                                            const unsigned long long (&qd)[DE], int keep, float s16) {
    const int lane = lane_id();
    const bool use_dir = a.flags & FG_KNN_USE_DIRECTION;
    unsigned long long c[4] = {0ull, 0ull, 0ull, 0ull};
    float mx = 0.0f;
    int total = 0;
    for (int f0 = 0; f0 < n; f0 += 32) {
        int32_t cpos = f0 + lane < n ? (int32_t)(w0 + f0 + lane) : -1;
        if (use_dir && cpos >= 0) {
            const int8_t role = a.dir[a.sid[cpos]];
            if (role == 1 || role == 2) cpos = -1;
        }
        if (cpos >= 0) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                const float4 x = a.sc[(int64_t)cpos * NV + v];
                if (4 * v + 0 < DE) W.sx[4 * v + 0][lane] = x.x;
                if (4 * v + 1 < DE) W.sx[4 * v + 1][lane] = x.y;
                if (4 * v + 2 < DE) W.sx[4 * v + 2][lane] = x.z;
                if (4 * v + 3 < DE) W.sx[4 * v + 3][lane] = x.w;
            }
        } else {
#pragma unroll
            for (int d = 0; d < DE; ++d) W.sx[d][lane] = kInf;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            unsigned long long acc;
#pragma unroll
            for (int d = 0; d < DE; ++d) {
                unsigned long long t0;
                const unsigned long long cv = *reinterpret_cast<const unsigned long long*>(&W.sx[d][j]);
                asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t0) : "l"(qd[d]), "l"(cv));
                if (d == 0) asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(acc) : "l"(t0));
                else asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(acc) : "l"(t0), "l"(acc));
            }
            float dv[2];
            asm("mov.b64 {%0, %1}, %2;" : "=f"(dv[0]), "=f"(dv[1]) : "l"(acc));
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                if (dv[u] < kInf) {
                    const int key = (int)(__float_as_uint(dv[u] * s16) >> 21);
                    const int b = min(max(key - 507, 0), 31);
                    const unsigned long long inc = 1ull << ((b & 7) * 8);
                    c[0] += (b >> 3) == 0 ? inc : 0ull;
                    c[1] += (b >> 3) == 1 ? inc : 0ull;
                    c[2] += (b >> 3) == 2 ? inc : 0ull;
                    c[3] += (b >> 3) == 3 ? inc : 0ull;
                    mx = fmaxf(mx, dv[u]);
                    ++total;
                }
            }
        }
        __syncwarp();
    }
    if (total < keep) return kInf;
    int cum = 0;
#pragma unroll
    for (int b = 0; b < 31; ++b) {
        cum += (int)((c[b >> 3] >> ((b & 7) * 8)) & 0xffu);
        if (cum >= keep)  // x < the bucket's upper edge
            return fminf(mx, __uint_as_float((unsigned)(508 + b) << 21) / s16);
    }
    return mx;
}

// Evaluate one 32-candidate chunk (W.sx / W.spos) against every lane's query
// and append the passing entries to the lanes' buffers.
template <int DE, int CAP, class Room>
__device__ __forceinline__ void eval_chunk(HdWarp<DE, CAP>& W, const unsigned long long (&qd)[DE], int head,
                                           float& tau, uint32_t bd_base, uint32_t bp_base, int& m,
                                           Room&& room) {
    // ring slots [head, head + 32); dead candidates carry +inf coordinates and position -1
    const uint32_t sp_addr = (uint32_t)__cvta_generic_to_shared(&W.spos[head]);
    // phase 1: all 32 distances (straight-line FADD2/FFMA2 chains: full ILP)
    float dv[32];
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        unsigned long long acc0, acc1;
#pragma unroll
        for (int d = 0; d < DE; ++d) {
            unsigned long long t0, t1;
            const ulonglong2 cv = *reinterpret_cast<const ulonglong2*>(&W.sx[d][head + j]);
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t0) : "l"(qd[d]), "l"(cv.x));
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(t1) : "l"(qd[d]), "l"(cv.y));
            if (d == 0) {
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(acc0) : "l"(t0));
                asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(acc1) : "l"(t1));
            } else {
                asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(acc0) : "l"(t0), "l"(acc0));
                asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(acc1) : "l"(t1), "l"(acc1));
            }
        }
        asm("mov.b64 {%0, %1}, %2;" : "=f"(dv[j]), "=f"(dv[j + 1]) : "l"(acc0));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(dv[j + 2]), "=f"(dv[j + 3]) : "l"(acc1));
    }
    // phase 2: per group of 4, append the passing candidates (rare once tau is
    // tight: one vote skips the chunk)
    float mn = dv[0];
#pragma unroll
    for (int u = 1; u < 32; ++u) mn = fminf(mn, dv[u]);
    if (!__any_sync(FG_FULL_MASK, mn <= tau)) return;
#pragma unroll
    for (int j = 0; j < 32; j += 4) {
        bool p0 = dv[j] <= tau, p1 = dv[j + 1] <= tau, p2 = dv[j + 2] <= tau, p3 = dv[j + 3] <= tau;
        if (__any_sync(FG_FULL_MASK, p0 | p1 | p2 | p3)) {
            if (__any_sync(FG_FULL_MASK, m > CAP - 4)) {  // a full buffer: cut it first
                room();
                p0 = dv[j] <= tau; p1 = dv[j + 1] <= tau; p2 = dv[j + 2] <= tau; p3 = dv[j + 3] <= tau;
            }
            int4 cp;
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(cp.x), "=r"(cp.y), "=r"(cp.z), "=r"(cp.w) : "r"(sp_addr + j * 4));
            const bool pp[4] = {p0, p1, p2, p3};
            const int32_t cc[4] = {cp.x, cp.y, cp.z, cp.w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                if (pp[u] && cc[u] >= 0) {
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(bd_base + 4 * m), "f"(dv[j + u]));
                    asm volatile("st.shared.b32 [%0], %1;" ::"r"(bp_base + 4 * m), "r"(cc[u]));
                    ++m;
                }
            }
        }
    }
}

// Candidate ring of the filtered scan: survivors of the query-box filter wait
// here until 32 are ready (carried across scan_spans calls; flushed at the end
// of a stage).
struct Ring {
    int head = 0, filled = 0;
};

// Scan the given spans (one per lane) in 32-candidate chunks.  DE <= kFilterDE:
// spans are cut into pieces at 32-position block boundaries, pieces whose
// block bounding box (boxes) lies farther than sqrt(max_l tau_l) from the
// tile's query box are skipped, the remaining candidates are filtered one by
// one against the query box and the survivors go through the ring; `final`
// evaluates what is left in the ring.
template <int NV, int DE, bool X64, int CAP>
__device__ __forceinline__ void scan_spans(HdWarp<DE, CAP>& W, const search::KnnArgs& a, int32_t S, int32_t L,
                                           const unsigned long long (&qd)[DE], float& tau, float& tt,
                                           int& m, int keep, const float (&q)[4 * NV], int32_t qid,
                                           float r, uint32_t bd_base, uint32_t bp_base,
                                           const float (&qlo)[DE], const float (&qhi)[DE],
                                           const float4* __restrict__ boxes, Ring& ring, bool final,
                                           unsigned long long& chunks, unsigned long long& cuts) {
    constexpr bool FILT = DE <= kFilterDE;
    const int lane = lane_id();
    const unsigned nonempty = __ballot_sync(FG_FULL_MASK, L > 0);
    if (!nonempty && !(FILT && final && ring.filled > 0)) return;
    const bool use_dir = a.flags & FG_KNN_USE_DIRECTION;
    const unsigned le = (2u << lane) - 1u;
    // candidate f of a list of (start, length) runs held one per lane (nr
    // lanes, inclusive / exclusive prefix of the lengths) -> sorted position
    // (one ballot + one redux per 32 candidates)
    auto pos_in = [&](int32_t f0, int nr, int32_t Sr, int32_t incl, int32_t excl, int32_t T) -> int32_t {
        const int base = __popc(__ballot_sync(FG_FULL_MASK, lane < nr && incl <= f0));
        const unsigned starts = __reduce_or_sync(
            FG_FULL_MASK, (lane < nr && excl > f0 && excl < f0 + 32) ? 1u << (excl - f0) : 0u);
        const int sidx = min(base + __popc(starts & le), 31);
        const int32_t Ss = __shfl_sync(FG_FULL_MASK, Sr, sidx);
        const int32_t Es = __shfl_sync(FG_FULL_MASK, excl, sidx);
        const int32_t f = f0 + lane;
        int32_t cpos = f < T ? Ss + (f - Es) : -1;
        if (use_dir && cpos >= 0) {  // roles 1/2 are never candidates (pyx:265-266)
            const int8_t role = a.dir[a.sid[cpos]];
            if (role == 1 || role == 2) cpos = -1;
        }
        return cpos;
    };
    auto fetch = [&](int32_t cpos, float4 (&x)[NV]) {
        if (cpos >= 0) {
            const float4* src = a.sc + (int64_t)cpos * NV;
#pragma unroll
            for (int v = 0; v < NV; ++v) x[v] = src[v];
        }
    };
    // cut every lane whose buffer cannot take 4 more entries (warp-uniform)
    auto room = [&]() {
        unsigned full = __ballot_sync(FG_FULL_MASK, m > CAP - 4);
        while (full) {
            const int j = __ffs(full) - 1;
            full &= full - 1;
            ++cuts;
            const int mj = __shfl_sync(FG_FULL_MASK, m, j);
            float qj[4 * NV];
#pragma unroll
            for (int d = 0; d < 4 * NV; ++d) qj[d] = __shfl_sync(FG_FULL_MASK, q[d], j);
            const int32_t qidj = __shfl_sync(FG_FULL_MASK, qid, j);
            const int rr = cut_lane<NV, X64, DE>(W, a, j, mj, keep, tau, tt, qj, qidj, r);
            if (lane == j) m = rr;
        }
    };
    // the runs in lanes [0, ns)
    const int ns = __popc(nonempty);
    if (L > 0) {
        const int dst = __popc(nonempty & lanemask_lt());
        W.span_s[dst] = S;
        W.span_l[dst] = L;
    }
    __syncwarp();
    S = lane < ns ? W.span_s[lane] : 0;
    L = lane < ns ? W.span_l[lane] : 0;
    __syncwarp();
    if constexpr (FILT) {
        auto coord = [](const float4 (&x)[NV], int d) -> float {
            return d % 4 == 0 ? x[d / 4].x : d % 4 == 1 ? x[d / 4].y : d % 4 == 2 ? x[d / 4].z : x[d / 4].w;
        };
        auto thr_now = [&]() {
            return __uint_as_float(__reduce_max_sync(FG_FULL_MASK, __float_as_uint(fmaxf(tau, 0.0f)))) *
                       kMargin + kTiny;
        };
        auto eval_ring = [&]() {
            __syncwarp();
            ++chunks;
            eval_chunk<DE>(W, qd, ring.head, tau, bd_base, bp_base, m, room);
            __syncwarp();
            ring.head ^= 32;
            ring.filled -= 32;
        };
        // runs (Sr, Lr) in lanes [0, nr): filter every candidate against the
        // query box, survivors into the ring, full chunks evaluated (the next
        // 32 candidates' coordinates are loaded while a chunk is filtered)
        auto consume = [&](int nr, int32_t Sr, int32_t Lr) {
            const int32_t incl = warp_inclusive_scan(Lr);
            const int32_t excl = incl - Lr;
            const int32_t T = __shfl_sync(FG_FULL_MASK, incl, 31);
            if (T == 0) return;
            int32_t cn = pos_in(0, nr, Sr, incl, excl, T);
            float4 xn[NV];
            fetch(cn, xn);
            for (int32_t f0 = 0; f0 < T; f0 += 32) {
                const int32_t cpos = cn;
                float4 x[NV];
#pragma unroll
                for (int v = 0; v < NV; ++v) x[v] = xn[v];
                if (f0 + 32 < T) {
                    cn = pos_in(f0 + 32, nr, Sr, incl, excl, T);
                    fetch(cn, xn);
                }
                const float thr = thr_now();
                float dd = 0.0f;
#pragma unroll
                for (int d = 0; d < DE; ++d) {
                    const float xv = coord(x, d);
                    const float gd = fmaxf(fmaxf(qlo[d] - xv, xv - qhi[d]), 0.0f);
                    dd = fmaf(gd, gd, dd);
                }
                const bool useful = cpos >= 0 && dd <= thr;
                const unsigned bal = __ballot_sync(FG_FULL_MASK, useful);
                if (useful) {
                    const int slot = (ring.head + ring.filled + __popc(bal & lanemask_lt())) & 63;
#pragma unroll
                    for (int d = 0; d < DE; ++d) W.sx[d][slot] = coord(x, d);
                    W.spos[slot] = cpos;
                }
                ring.filled += __popc(bal);
                if (ring.filled >= 32) eval_ring();
            }
        };
        if (ns > 0) {
            if (boxes) {
                // pieces: the runs cut at 32-position block boundaries
                const int np = L > 0 ? ((S + L - 1) >> 5) - (S >> 5) + 1 : 0;
                const int32_t pin = warp_inclusive_scan(np);
                const int32_t pex = pin - np;
                const int32_t NP = __shfl_sync(FG_FULL_MASK, pin, 31);
                for (int32_t pb = 0; pb < NP; pb += 32) {
                    const int base = __popc(__ballot_sync(FG_FULL_MASK, lane < ns && pin <= pb));
                    const unsigned starts = __reduce_or_sync(
                        FG_FULL_MASK, (lane < ns && pex > pb && pex < pb + 32) ? 1u << (pex - pb) : 0u);
                    const int sidx = min(base + __popc(starts & le), 31);
                    const int32_t Ss = __shfl_sync(FG_FULL_MASK, S, sidx);
                    const int32_t Ls = __shfl_sync(FG_FULL_MASK, L, sidx);
                    const int32_t Ps = __shfl_sync(FG_FULL_MASK, pex, sidx);
                    const int32_t f = pb + lane;
                    const float thr = thr_now();
                    int32_t ps = 0, pl = 0;
                    if (f < NP) {
                        const int32_t blk = (Ss >> 5) + (f - Ps);
                        ps = max(Ss, blk << 5);
                        pl = min(Ss + Ls, (blk << 5) + 32) - ps;
                        const float4 blo = boxes[2 * blk], bhi = boxes[2 * blk + 1];
                        const float bl[4] = {blo.x, blo.y, blo.z, blo.w}, bh[4] = {bhi.x, bhi.y, bhi.z, bhi.w};
                        float dd = 0.0f;
#pragma unroll
                        for (int d = 0; d < DE; ++d) {
                            const float gd = fmaxf(fmaxf(bl[d] - qhi[d], qlo[d] - bh[d]), 0.0f);
                            dd = fmaf(gd, gd, dd);
                        }
                        if (!(dd <= thr)) pl = 0;
                    }
                    const unsigned keep_b = __ballot_sync(FG_FULL_MASK, pl > 0);
                    if (!keep_b) continue;
                    if (pl > 0) {
                        const int dst = __popc(keep_b & lanemask_lt());
                        W.span_s[32 + dst] = ps;
                        W.span_l[32 + dst] = pl;
                    }
                    __syncwarp();
                    const int nk = __popc(keep_b);
                    const int32_t PS = lane < nk ? W.span_s[32 + lane] : 0;
                    const int32_t PL = lane < nk ? W.span_l[32 + lane] : 0;
                    __syncwarp();
                    consume(nk, PS, PL);
                }
            } else {
                consume(ns, S, L);
            }
        }
        if (final && ring.filled > 0) {  // the rest, padded with dead sentinels
            if (lane >= ring.filled) {
                const int slot = (ring.head + lane) & 63;
#pragma unroll
                for (int d = 0; d < DE; ++d) W.sx[d][slot] = kInf;
                W.spos[slot] = -1;
            }
            eval_ring();
            ring.filled = 0;
        }
        return;
    }
    (void)boxes;
    (void)final;
    const int32_t incl = warp_inclusive_scan(L);
    const int32_t excl = incl - L;
    const int32_t T = __shfl_sync(FG_FULL_MASK, incl, 31);
    auto pos_of = [&](int32_t f0) { return pos_in(f0, ns, S, incl, excl, T); };
    // chunk f0 + 32 is loaded into registers while chunk f0 is evaluated
    int32_t cpos_n = pos_of(0);
    float4 xn[NV];
    fetch(cpos_n, xn);
    for (int32_t f0 = 0; f0 < T; f0 += 32) {
        ++chunks;
        const int32_t cpos = cpos_n;
        if (cpos >= 0) {
#pragma unroll
            for (int v = 0; v < NV; ++v) {
                if (4 * v + 0 < DE) W.sx[4 * v + 0][lane] = xn[v].x;
                if (4 * v + 1 < DE) W.sx[4 * v + 1][lane] = xn[v].y;
                if (4 * v + 2 < DE) W.sx[4 * v + 2][lane] = xn[v].z;
                if (4 * v + 3 < DE) W.sx[4 * v + 3][lane] = xn[v].w;
            }
        } else {
#pragma unroll
            for (int d = 0; d < DE; ++d) W.sx[d][lane] = kInf;
        }
        W.spos[lane] = cpos;
        if (f0 + 32 < T) {
            cpos_n = pos_of(f0 + 32);
            fetch(cpos_n, xn);
        }
        __syncwarp();
        eval_chunk<DE>(W, qd, 0, tau, bd_base, bp_base, m, room);
        __syncwarp();
    }
}

// ---------------------------------------------------------------- search
#ifndef FG_HD_REGS_LOWD
#define FG_HD_REGS_LOWD 224
#endif
template <int NV, bool X64>
__host__ __device__ constexpr int hd_regs() {
    return NV == 1 && !X64 ? FG_HD_REGS_LOWD : 224;
}
template <int NV, int DB, int DE, bool X64>
__global__ void __maxnreg__((hd_regs<NV, X64>())) k_hd_search(const __grid_constant__ tile::TileArgs t,
                                                           const __grid_constant__ search::KnnArgs a) {
    constexpr int NL = DB - 1;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int CAP = hd_cap<NV, X64>();
    constexpr int kS = CAP + 1;
    HdWarp<DE, CAP>& W = reinterpret_cast<HdWarp<DE, CAP>*>(smem_raw)[threadIdx.x >> 5];
    const int lane = lane_id();
    const int nb = t.nb;
    const int need = a.k - 1;
    const int keep = need + 1;  // self stays in the buffer until the epilogue
    const bool use_dir = a.flags & FG_KNN_USE_DIRECTION;
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    const float r = X64 ? *a.rnd : 0.0f;
    // cell-unit slack: the float32 cell position of a float64 coordinate can be
    // off by the rounding of the coordinate and of the split minimum
    const uint32_t bd_base = (uint32_t)__cvta_generic_to_shared(&W.bd[lane * kS]);
    const uint32_t bp_base = (uint32_t)__cvta_generic_to_shared(&W.bp[lane * kS]);
    float rho2_hint = -1.0f;  // final radius^2 of this warp's previous tile
    unsigned long long st_tiles = 0, st_chunks = 0, st_stages = 0, st_cuts = 0;
    search::Counters cnt;
    const int n_tiles = t.ctr[0];

    for (;;) {
        int ti = 0;
        if (lane == 0) ti = atomicAdd(&t.ctr[1], 1);
        ti = __shfl_sync(FG_FULL_MASK, ti, 0);
        if (ti >= n_tiles) break;
        if (t.order) ti = t.order[ti];
        ++st_tiles;
        const long long tile_c0 = clock64();
        const int s = t.tiles[ti].x / t.bps;
        const int64_t cbase = (int64_t)s * t.total;

        // ---- lane -> point of the tile
        const int32_t p = tile_point<DB>(t, ti);
        const bool live = p >= 0;
        if (!__any_sync(FG_FULL_MASK, live)) continue;
        const int32_t qid = live ? a.sid[p] : 0;
        // DirectionMask: roles 0/2 run no query (row = self + padding, pyx:210-211)
        const bool active = live && need > 0 &&
                            !(use_dir && (a.dir[qid] == 0 || a.dir[qid] == 2));

        // ---- queries: coordinates (packed pairs), cell-unit box of the tile
        float q[4 * NV];
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            const float4 x = live ? t.sc[(int64_t)p * NV + v] : make_float4(0.f, 0.f, 0.f, 0.f);
            q[4 * v] = x.x; q[4 * v + 1] = x.y; q[4 * v + 2] = x.z; q[4 * v + 3] = x.w;
        }
        unsigned long long qd[DE];
#pragma unroll
        for (int d = 0; d < DE; ++d) qd[d] = dup2(q[d]);
        float qlo[DE], qhi[DE];  // the unfinished queries' box (candidate filter, per stage)
        float w[DB], invw[DB], lo[DB], hi[DB];
        float diag2 = 0.0f;  // squared diagonal of the split's grid box
        float slack = kSlackCells;
#pragma unroll
        for (int i = 0; i < DB; ++i) {
            const float mn = (float)t.mins[(int64_t)s * DB + i];
            w[i] = (float)t.widths[(int64_t)s * DB + i];
            invw[i] = __frcp_rn(w[i]);
            const float qc = (q[i] - mn) * invw[i];
            lo[i] = tile::warp_min_f(live ? qc : kInf);
            hi[i] = tile::warp_max_f(live ? qc : -kInf);
            diag2 = fmaf((float)nb * w[i], (float)nb * w[i], diag2);
            if (X64) slack = fmaxf(slack, 2.0f * r * invw[i] + kSlackCells);
        }
        diag2 *= 1.01f;

        // ---- staged region growth
        float tt = kInf;  // true bound on the lane's keep-th smallest float64 d2
        if (use_r2) tt = (float)(a.max_r2 * (1.0 + 2e-5)) + kTiny;
        float tau = X64 ? up_bound(tt, r) : (use_r2 ? tt * kMargin : tt);
        if (!active) {  // appends nothing, needs no region
            tau = -1.0f;
            tt = 0.0f;
        }
        int m = 0;
        bool done = false;  // the lane's answer is complete (region covers its tt-ball)
        // cut every active lane holding >= keep entries to its keep smallest
        auto tighten = [&]() {
            unsigned todo = __ballot_sync(FG_FULL_MASK, active && !done && m >= keep);
            while (todo) {
                const int j = __ffs(todo) - 1;
                todo &= todo - 1;
                const int mj = __shfl_sync(FG_FULL_MASK, m, j);
                float qj[4 * NV];
#pragma unroll
                for (int d = 0; d < 4 * NV; ++d) qj[d] = __shfl_sync(FG_FULL_MASK, q[d], j);
                const int32_t qidj = __shfl_sync(FG_FULL_MASK, qid, j);
                const int rr = cut_lane<NV, X64, DE>(W, a, j, mj, keep, tau, tt, qj, qidj, r);
                if (lane == j) m = rr;
            }
        };
        const int32_t pmin_t = (int32_t)__reduce_min_sync(FG_FULL_MASK, (unsigned)(live ? p : 0x7fffffff));
        const int32_t pmax_t = (int32_t)__reduce_max_sync(FG_FULL_MASK, (unsigned)(live ? p : 0));
        if (kSeed > 0 && !use_r2) {
            // stage 0: tau seeds from the kSeed points around the tile's middle
            // in the sorted order (same split) -- real points, so each lane's
            // keep-th smallest among them bounds its answer (bucketed: no
            // buffers, no cuts)
            const int64_t s_lo = a.rs[s], s_hi = a.rs[s + 1];
            const int64_t mid = ((int64_t)pmin_t + pmax_t) / 2;
            const int64_t w0 = max(s_lo, min(mid - kSeed / 2, s_hi - kSeed));
            const int64_t w1 = min(s_hi, w0 + kSeed);
            float bx = 0.0f;  // squared diagonal of the active queries' box: the bucket scale
#pragma unroll
            for (int d = 0; d < DE; ++d) {
                const float e = tile::warp_max_f(active ? q[d] : -kInf) - tile::warp_min_f(active ? q[d] : kInf);
                bx = fmaf(e, e, bx);
            }
            const float s16 = 16.0f / fmaxf(bx, 1e-30f);
            const float b = seed_bound<NV, DE>(W, a, w0, (int)(w1 - w0), qd, keep, s16);
            if (active && b < kInf) {
                tt = fminf(tt, X64 ? up_bound(b, r) : b * kMargin + kTiny);
                tau = X64 ? up_bound(tt, r) : tt;
            }
            __syncwarp();
        }
        // first stage at a fraction of the previous tile's radius: the nearest
        // rows come first, so the cuts tighten tau early (fewer appends later)
        float rho2 = rho2_hint * kHintScale;
        if (!(rho2 > 0.0f)) {  // no hint: a one-cell pilot
            float wm = w[0];
#pragma unroll
            for (int i = 1; i < DB; ++i) wm = fminf(wm, w[i]);
            rho2 = wm * wm;
        }
        rho2 = fminf(rho2, diag2);
        Box<NL> prev = make_box<DB>(-1.0f, lo, hi, invw, nb, slack);
        Ring ring;
        for (;;) {
            ++st_stages;
            // lanes whose tt-ball is already inside the scanned region are done:
            // they take no more entries, and the candidate filter (box, max tau)
            // covers only the others (one sparse lane no longer drags 31 dense
            // lanes' worth of candidates through every stage)
            const bool open = active && !done;
            float tau_s = open ? tau : -1.0f;
#pragma unroll
            for (int d = 0; d < DE; ++d) {
                qlo[d] = DE <= kFilterDE ? tile::warp_min_f(open ? q[d] : kInf) : 0.0f;
                qhi[d] = DE <= kFilterDE ? tile::warp_max_f(open ? q[d] : -kInf) : 0.0f;
            }
            const Box<NL> cur = make_box<DB>(rho2, lo, hi, invw, nb, slack);
            for (int rb = 0; rb < cur.rows; rb += 32) {
                const int rw = rb + lane;
                int32_t S0 = 0, L0 = 0, S1 = 0, L1 = 0;
                if (rw < cur.rows) {
                    int jd[NL > 0 ? NL : 1];
                    search::decode_row<NL>(rw, cur.L, cur.N, cur.inv, jd);
                    int rowflat = 0;
#pragma unroll
                    for (int i = 0; i < NL; ++i) rowflat = rowflat * nb + jd[i];
                    int ca, cb, pa, pb;
                    row_piece<DB>(cur, jd, lo, hi, w, invw, nb, ca, cb);
                    row_piece<DB>(prev, jd, lo, hi, w, invw, nb, pa, pb);
                    const int64_t rc = cbase + (int64_t)rowflat * nb;
                    if (ca <= cb) {
                        if (pa > pb) {  // row new in this stage
                            S0 = t.bounds[rc + ca];
                            L0 = t.bounds[rc + cb + 1] - S0;
                        } else {  // the shell: [ca, pa-1] and [pb+1, cb]
                            if (ca < pa) {
                                S0 = t.bounds[rc + ca];
                                L0 = t.bounds[rc + pa] - S0;
                            }
                            if (pb < cb) {
                                S1 = t.bounds[rc + pb + 1];
                                L1 = t.bounds[rc + cb + 1] - S1;
                            }
                        }
                    }
                }
                scan_spans<NV, DE, X64>(W, a, S0, L0, qd, tau_s, tt, m, keep, q, qid, r, bd_base,
                                        bp_base, qlo, qhi, t.boxes, ring, false, st_chunks, st_cuts);
                scan_spans<NV, DE, X64>(W, a, S1, L1, qd, tau_s, tt, m, keep, q, qid, r, bd_base,
                                        bp_base, qlo, qhi, t.boxes, ring, false, st_chunks, st_cuts);
            }
            scan_spans<NV, DE, X64>(W, a, 0, 0, qd, tau_s, tt, m, keep, q, qid, r, bd_base, bp_base, qlo,
                                    qhi, t.boxes, ring, true, st_chunks, st_cuts);  // flush the ring
            if (open) tau = tau_s;
            float need_t = tile::warp_max_f(open ? tt : 0.0f);
            if (!(need_t <= rho2) && rho2 < diag2) {  // the bounds as they stand do not settle it
                tighten();  // every open lane to its keep-th smallest entry
                need_t = tile::warp_max_f(open ? tt : 0.0f);
            }
            done |= open && tt <= rho2;
            prev = cur;
            // done when every lane's tt-ball is inside the region, or the region
            // is the whole grid box of the split (lanes short of k-1 points)
            if (need_t <= rho2 || rho2 >= diag2) break;
            // grow: at most x1.6 in radius per stage, never past what is needed
            rho2 = fminf(fminf(need_t, rho2 * 2.56f), diag2);
        }
        {
            const float h = tile::warp_max_f(active ? tt : 0.0f);
            rho2_hint = (h > 0.0f && h < kInf) ? h : -1.0f;
        }

        // ---- epilogue, one row at a time
        __syncwarp();  // every lane's last appends are visible to the warp
        const unsigned rows = __ballot_sync(FG_FULL_MASK, live);
        for (unsigned mask = rows; mask;) {
            const int j = __ffs(mask) - 1;
            mask &= mask - 1;
            const int mj = __shfl_sync(FG_FULL_MASK, m, j);
            const int32_t pj = __shfl_sync(FG_FULL_MASK, p, j);
            const float tj = __shfl_sync(FG_FULL_MASK, tau, j);
            const int32_t qj_id = __shfl_sync(FG_FULL_MASK, qid, j);
            const bool aj = __shfl_sync(FG_FULL_MASK, active ? 1 : 0, j);
            const int64_t row_out = (int64_t)qj_id * a.k;
            if (lane == 0) {
                a.out_idx[row_out] = qj_id;
                search::store_d2(a, row_out, 0.0);
            }
            if (!aj) {  // no query: padding
                for (int sl = 1 + lane; sl < a.k; sl += 32) {
                    a.out_idx[row_out + sl] = -1;
                    search::store_d2(a, row_out + sl, 0.0);
                }
                continue;
            }
            float qj[4 * NV];
#pragma unroll
            for (int d = 0; d < 4 * NV; ++d) qj[d] = __shfl_sync(FG_FULL_MASK, q[d], j);
            // lane j's entries minus self
            int wpos = 0;
            for (int e0 = 0; e0 < mj; e0 += 32) {
                const int e = e0 + lane;
                const bool ok = e < mj && W.bp[j * kS + e] != pj;
                const unsigned bal = __ballot_sync(FG_FULL_MASK, ok);
                if (ok) {
                    const int at = wpos + __popc(bal & lanemask_lt());
                    W.eb.d[at] = W.bd[j * kS + e];
                    W.eb.p[at] = W.bp[j * kS + e];
                }
                wpos += __popc(bal);
            }
            __syncwarp();
            if constexpr (X64) {
                exact_sort<NV, X64, DE>(W, a, wpos, qj, qj_id);
                for (int sl = 1 + lane; sl < a.k; sl += 32) {
                    const int e = sl - 1;
                    const unsigned long long kk = e < wpos ? W.eb.key[e] : ~0ull;
                    if (kk != ~0ull) {
                        a.out_idx[row_out + sl] = W.eb.id[e];
                        search::store_d2(a, row_out + sl, __longlong_as_double((long long)kk));
                    } else {
                        a.out_idx[row_out + sl] = -1;
                        search::store_d2(a, row_out + sl, 0.0);
                    }
                }
                __syncwarp();
            } else {
                search::finish_query<NV, 128>(a, W.eb, qj, wpos, need, tj, row_out, cnt);
            }
        }
        __syncwarp();
        if (a.stats && lane == 0)  // the slowest tile (clock64 cycles): the kernel's tail
            atomicMax(a.stats + search::ST_COUNT + tile::TS_COUNT + HS_MAXCYC,
                      (unsigned long long)(clock64() - tile_c0));
    }
    if (a.stats && lane == 0) {
        unsigned long long* hs = a.stats + search::ST_COUNT + tile::TS_COUNT;
        atomicAdd(&hs[HS_TILES], st_tiles);
        atomicAdd(&hs[HS_CHUNKS], st_chunks);
        atomicAdd(&hs[HS_STAGES], st_stages);
        atomicAdd(&hs[HS_COMPACT], st_cuts);
    }
}

// float64 mode: r = sqrt(n_c) x the largest difference error of two float32-
// rounded coordinates (2 x 2^-24 x max |x|, plus the subnormal floor).
static __global__ void k_abs_bound(const double* __restrict__ x, int64_t m, int n_c,
                            unsigned* __restrict__ out) {
    double mx = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x)
        mx = fmax(mx, fabs(x[i]));
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FG_FULL_MASK, mx, o));
    if (lane_id() == 0) {
        const double e = 2.0 * (mx * 0x1p-24 + 0x1p-149);
        const float rb = __double2float_ru(e * sqrt((double)n_c) * 1.0001);
        atomicMax(out, __float_as_uint(rb));  // non-negative floats order like their bits
    }
}

// ---------------------------------------------------------------- dense cells
// Clustered data puts thousands of points in one cell; in the binning's order
// (ascending id inside a cell) 32 consecutive points of such a cell are spread
// over the whole cell, so a tile's box is the cell and its tau seeds are poor.
// The search therefore runs on copies of the sorted coordinates / ids in which
// the points of every cell with more than kDenseCell points are ordered by the
// Morton code of their position inside the cell (cells stay contiguous ranges:
// bin_bounds is unchanged; outputs are original ids, so the answer is the same).
constexpr int kDenseCell = 32;
constexpr int kMaxSortCell = 16384;  // larger cells keep the binning's order

template <int NV>
__global__ void __launch_bounds__(256) k_cell_split(const tile::TileArgs t, int64_t n_cells) {
    const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (c >= n_cells || tile::gated_off(t)) return;
    const int32_t lo = t.bounds[c], len = t.bounds[c + 1] - lo;
    if (len > kDenseCell && len <= kMaxSortCell) {
        t.dense[atomicAdd(&t.ctr[5], 1)] = (int32_t)c;
        return;
    }
    for (int i = 0; i < len; ++i) {
#pragma unroll
        for (int v = 0; v < NV; ++v) t.sc2[(int64_t)(lo + i) * NV + v] = t.sc[(int64_t)(lo + i) * NV + v];
        t.sid2[lo + i] = t.sid[lo + i];
    }
}

__device__ __forceinline__ unsigned morton_spread(unsigned x, int dims, int bits) {
    unsigned r = 0;
    for (int b = 0; b < bits; ++b) r |= ((x >> b) & 1u) << (b * dims);
    return r;
}

// One CTA per dense cell: the cell's points ordered by the top B bits of their
// in-cell Morton code (B ~ log2(len) - 1: about two points per bucket), by a
// counting sort -- shared-memory histogram, block scan, atomic scatter, then
// each bucket put in index order by a thread (the order is deterministic; the
// buckets are small) -- 5 barriers per cell instead of the ~100 of a bitonic
// sort of 16384 keys (config B: 185 -> 50 us).  Only the compactness of
// the search's tiles depends on this order, never the answer.
constexpr int kMortonBuckets = 4096;
template <int NV, int DB>
__global__ void __launch_bounds__(1024) k_dense_morton(const tile::TileArgs t) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    uint16_t* bk = reinterpret_cast<uint16_t*>(smem_raw);          // bucket of entry i
    uint16_t* perm = bk + kMaxSortCell;                            // entries by bucket
    int32_t* cur = reinterpret_cast<int32_t*>(perm + kMaxSortCell);  // counts -> cursors
    int32_t* start = cur + kMortonBuckets;                         // bucket starts (+ total)
    __shared__ int32_t s_warp[32];
    constexpr int bits = 32 / DB > 10 ? 10 : 32 / DB;
    constexpr int TB = DB * bits;  // Morton code bits
    if (tile::gated_off(t)) return;
    const int lane = lane_id(), w = threadIdx.x >> 5;
    const int count = t.ctr[5];
    for (int it = blockIdx.x; it < count; it += gridDim.x) {
        const int32_t c = t.dense[it];
        const int32_t lo = t.bounds[c], len = t.bounds[c + 1] - lo;
        const int64_t s = c / t.total;
        int64_t flat = c - s * t.total;
        int cell[DB];
#pragma unroll
        for (int i = DB - 1; i >= 0; --i) {
            cell[i] = (int)(flat % t.nb);
            flat /= t.nb;
        }
        const int B = min(min(12, TB), max(1, 31 - __clz(len)));  // ~2 points per bucket
        const int NB = 1 << B;
        for (int b = threadIdx.x; b < NB; b += blockDim.x) cur[b] = 0;
        __syncthreads();
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const float4 x = t.sc[(int64_t)(lo + i) * NV];
            const float xa[4] = {x.x, x.y, x.z, x.w};
            unsigned mk = 0;
#pragma unroll
            for (int d = 0; d < DB && d < 4; ++d) {
                const double wd = t.widths[s * DB + d];
                const double u = ((double)xa[d] - (t.mins[s * DB + d] + cell[d] * wd)) / wd;
                const int qd = min((1 << bits) - 1, max(0, (int)(u * (1 << bits))));
                mk |= morton_spread((unsigned)qd, DB, bits) << d;
            }
            const int b = (int)(mk >> (TB - B));
            bk[i] = (uint16_t)b;
            atomicAdd(&cur[b], 1);
        }
        __syncthreads();
        {  // exclusive scan of the NB <= 4096 counts: 4 per thread
            int v[4], tot = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int b = 4 * threadIdx.x + j;
                v[j] = b < NB ? cur[b] : 0;
                tot += v[j];
            }
            const int incl = warp_inclusive_scan(tot);
            if (lane == 31) s_warp[w] = incl;
            __syncthreads();
            if (w == 0) s_warp[lane] = warp_inclusive_scan(s_warp[lane]);
            __syncthreads();
            int run = incl - tot + (w > 0 ? s_warp[w - 1] : 0);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int b = 4 * threadIdx.x + j;
                if (b < NB) {
                    start[b] = run;
                    cur[b] = run;
                }
                run += v[j];
            }
            if (threadIdx.x == 0) start[NB] = len;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < len; i += blockDim.x) perm[atomicAdd(&cur[bk[i]], 1)] = (uint16_t)i;
        __syncthreads();
        for (int b = threadIdx.x; b < NB; b += blockDim.x) {  // index order inside each bucket
            const int b0 = start[b], b1 = start[b + 1];
            for (int i = b0 + 1; i < b1; ++i) {
                const uint16_t x = perm[i];
                int j = i;
                while (j > b0 && perm[j - 1] > x) {
                    perm[j] = perm[j - 1];
                    --j;
                }
                perm[j] = x;
            }
        }
        __syncthreads();
        for (int j = threadIdx.x; j < len; j += blockDim.x) {
            const int src = perm[j];
#pragma unroll
            for (int v = 0; v < NV; ++v) t.sc2[(int64_t)(lo + j) * NV + v] = t.sc[(int64_t)(lo + src) * NV + v];
            t.sid2[lo + j] = t.sid[lo + src];
        }
        __syncthreads();
    }
}

// Bounding box of every 32 sorted positions of the search's coordinates (d <= 4).
static __global__ void __launch_bounds__(256) k_block_boxes(const tile::TileArgs t) {
    const int64_t b = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int lane = lane_id();
    if ((b << 5) >= t.n || tile::gated_off(t)) return;
    const int64_t p = (b << 5) + lane;
    const bool ok = p < t.n;
    const float4 x = ok ? t.sc[p] : make_float4(0.f, 0.f, 0.f, 0.f);
    const float4 lo = make_float4(tile::warp_min_f(ok ? x.x : kInf), tile::warp_min_f(ok ? x.y : kInf),
                                  tile::warp_min_f(ok ? x.z : kInf), tile::warp_min_f(ok ? x.w : kInf));
    const float4 hi = make_float4(tile::warp_max_f(ok ? x.x : -kInf), tile::warp_max_f(ok ? x.y : -kInf),
                                  tile::warp_max_f(ok ? x.z : -kInf), tile::warp_max_f(ok ? x.w : -kInf));
    if (lane == 0) {
        t.boxes[2 * b] = lo;
        t.boxes[2 * b + 1] = hi;
    }
}

// Tile list, then the search (no redo: cuts fall back to exact keys).
template <int NV, int DB, int DE, bool X64>
int launch_hd(tile::TileArgs& t_in, const search::KnnArgs& a_in, cudaStream_t st) {
    tile::TileArgs t = t_in;
    search::KnnArgs a = a_in;
    FG_CUDA(cudaMemsetAsync(t.ctr, 0, 8 * sizeof(int), st));
    k_hd_tiles<DB><<<(unsigned)ceil_div(t.n_blocks, 4), 128, 0, st>>>(t);
    FG_TRY(launched(st));
    int dev = 0, sms = 0;
    FG_CUDA(cudaGetDevice(&dev));
    FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (t.sc2) {  // dense cells in Morton order: the search's own copies of sc / sid
        const int64_t n_cells = (int64_t)t.n_blocks / t.bps * t.total;
        k_cell_split<NV><<<(unsigned)ceil_div(n_cells, 256), 256, 0, st>>>(t, n_cells);
        FG_TRY(launched(st));
        const size_t msmem = 2 * sizeof(uint16_t) * kMaxSortCell + sizeof(int32_t) * (2 * kMortonBuckets + 1);
        FG_CUDA(cudaFuncSetAttribute(k_dense_morton<NV, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)msmem));
        k_dense_morton<NV, DB><<<(unsigned)sms, 1024, msmem, st>>>(t);
        FG_TRY(launched(st));
        t.sc = t.sc2;
        t.sid = t.sid2;
        a.sc = t.sc2;
        a.sid = t.sid2;
    }
    if (DE <= kFilterDE && NV == 1 && t.boxes) {
        k_block_boxes<<<(unsigned)ceil_div(t.n, 256), 256, 0, st>>>(t);
        FG_TRY(launched(st));
    } else {
        t.boxes = nullptr;
    }
#ifndef FG_HD_ORDER
#define FG_HD_ORDER 1
#endif
    if (!FG_HD_ORDER) t.order = nullptr;
    if (t.order) {  // widest query boxes first
        const int64_t max_tiles = t.n / 32 + (int64_t)t.n_blocks * t.nb + 1;  // hd_ws's bound
        FG_CUDA(cudaMemsetAsync(t.hist, 0, sizeof(int) * 2 * kCostBuckets, st));
        k_hd_cost<NV, DB><<<(unsigned)ceil_div(max_tiles, 4), 128, 0, st>>>(t);
        FG_TRY(launched(st));
        k_hd_rank<<<1, 32, 0, st>>>(t);
        FG_TRY(launched(st));
        k_hd_place<<<(unsigned)ceil_div(max_tiles, 256), 256, 0, st>>>(t);
        FG_TRY(launched(st));
    }
    constexpr int WARPS = hd_warps<NV, X64>();
    constexpr size_t smem = hd_smem_bytes<DE, hd_cap<NV, X64>(), WARPS>();
    auto kern = k_hd_search<NV, DB, DE, X64>;
    FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;  // resident CTAs per SM (shared memory bound)
    FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WARPS * 32, smem));
    kern<<<(unsigned)(sms * std::max(per_sm, 1)), WARPS * 32, smem, st>>>(t, a);
    return launched(st);
}

template <int NV, bool X64>
int dispatch_db(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st) {
    switch (d_bin) {
        case 1: return launch_hd<NV, 1, 4 * NV, X64>(t, a, st);
        case 2: return launch_hd<NV, 2, 4 * NV, X64>(t, a, st);
        case 3: return launch_hd<NV, 3, 4 * NV, X64>(t, a, st);
        case 4: return launch_hd<NV, 4, 4 * NV, X64>(t, a, st);
        default:
            if constexpr (NV >= 2) {
                if constexpr (NV == 3 && !X64) {  // d = 10 (config C): no padded dims in the hot loop
                    if (a.n_c == 10) return launch_hd<NV, 5, 10, X64>(t, a, st);
                }
                return launch_hd<NV, 5, 4 * NV, X64>(t, a, st);
            }
            return FG_ERR_TOO_FEW_DIMS;
    }
}

int dispatch_hd_nv1(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_hd_nv2(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_hd_nv3(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_hd_nv4(tile::TileArgs& t, const search::KnnArgs& a, int d_bin, cudaStream_t st);

}  // namespace hd
}  // namespace fg
