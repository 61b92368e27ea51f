// fg_knn_impl.cuh -- binned_select_knn forward for sm_100a (replaces pyx:188-329).
//
// One warp per query; queries are visited in sorted (cell-major) order so the
// warps resident on an SM read overlapping candidate rows through L1/L2.
// Templated on NV (float4 vectors per point), DB (binned dims, 1..5) and CAP
// (candidate buffer entries per warp).
//
// Per query q (sorted position p, original id qid, cell c, grid position qc in
// cell units):
//  * regions.  The search scans nested Chebyshev cubes around c:
//    region (R_old, R_new] = cube(R_new) minus cube(R_old).  A "row" is a fixed
//    choice of the leading DB-1 cells; along the last binned dim a row of cells
//    is ONE contiguous span of sorted points (flat ids are row-major,
//    G/stepper.py:20-31), so a row contributes one span (two when the row
//    passes through the already-scanned cube).  Lane r owns row r: it prunes
//    the row by its lead-dim box distance to q against tau and trims the span
//    to the cells the tau-ball reaches.
//  * flattening.  The non-empty spans of a 32-row batch are compacted to lanes
//    0..n-1, prefix-summed, and every 32-candidate chunk is mapped back to its
//    span with one ballot + one redux.sync.or.
//  * filter.  d2 = sum (q_i - x_i)^2 in fp32; a candidate enters the warp's
//    shared-memory buffer iff d2 <= tau (self, hidden roles and max_radius2
//    applied here).  compact() radix-selects an upper bound T of the (k-1)-th
//    smallest buffered d2; tau = T*(1+1e-5) and everything above it is dropped.
//  * speculative radius.  When every coordinate is binned, tau0 = (1.1 x the
//    k-th-neighbour distance expected from the density of the 3^DB cube around
//    c)^2 and the first region is the cube covering the tau0-ball, pruned and
//    filtered at tau0.  If >= k-1 neighbours lie strictly inside tau0 (with a
//    3e-5 margin) the answer is certified; otherwise the query restarts plainly.
//  * certificate.  After a region the next one is the smallest cube covering
//    the tau-ball around q (per query, from its own position); when it is not
//    larger than what was scanned nothing unscanned can reach the answer -- the
//    reference's (w_min*r)^2 > maxd2 stop (pyx:288-296) made per query and per
//    dimension.
//  * exact epilogue.  Buffered candidates get their float64 d2 recomputed in the
//    reference's operation order (pyx:32-48, no FMA).  Fast path: a register
//    bitonic sort (64 or 128 keys) on (float32(d2_f64) bits, position); if two
//    entries that decide the row share a float32 value (ties / sub-ulp
//    near-ties) the exact path runs instead: a shared-memory sort on
//    (d2_f64, original index).  Rows come out sorted by (d2_f64, original index)
//    -- lower index wins exact ties -- with slot 0 = self and (-1, 0) padding.
//    fp32 d2 is within ~1e-6 relative of the float64 value and every filter
//    keeps a >= 1e-5 margin, so the answer equals the float64 canonical answer
//    bit for bit.
#pragma once
#include <cfloat>

#ifndef FG_SPAN_WALK
#define FG_SPAN_WALK 0
#endif
#ifndef FG_EPI_BITONIC
#define FG_EPI_BITONIC 0
#endif
#ifndef FG_EPI_CUT
#define FG_EPI_CUT 64
#endif
#ifndef FG_ALPHA
#define FG_ALPHA 1.07f
#endif
#ifndef FG_KNN_MINB
#define FG_KNN_MINB 8
#endif

#include "fg_common.cuh"

namespace fg {
namespace search {

constexpr int kWarpsPerBlock = 4;
constexpr float kMargin = 1.0f + 1e-5f;
constexpr float kTiny = 1e-35f;
constexpr float kCellSlack = 1e-4f;  // cell units
constexpr float kAlpha = FG_ALPHA;   // speculative radius inflation
constexpr float kInf = __builtin_huge_valf();

enum { ST_QUERIES, ST_REGIONS, ST_CHUNKS, ST_APPENDS, ST_COMPACT, ST_SPEC_FAIL, ST_EXACT_EPI,
       ST_ROWS, ST_COUNT };

struct KnnArgs {
    const float4* sc;  // sorted coords, NV float4 per point
    const int32_t* sid;
    const int64_t* bin_idx;
    const int32_t* bounds;
    const int64_t* rs;
    const double* mins;
    const double* widths;
    int64_t n;
    int64_t total;
    int n_c, n_splits, nb, k;
    const int8_t* dir;
    double max_r2;
    uint32_t flags;
    int32_t* out_idx;
    void* out_d2;
    unsigned long long* stats;  // device counters (FG_KNN_STATS) or null
    const int32_t* qlist;       // optional query list (sorted positions), e.g. the
    const int* qcount;          // tile path's redo list; its length lives on the device
    const int* qall;            // with qlist: *qall * 4 > n -> every query instead (the
                                // tile kernels declined the data, fg_knn_tile.cuh)
    const double* x64;          // float64 coordinates (original order, n x n_c) or null:
                                // exact keys from them (fg_knn_hd.cuh float64 mode)
    const float* rnd;           // float64 mode: device bound on |fp32 - float64| coordinate
                                // differences x sqrt(n_c) (k_abs_bound)
};

template <int CAP>
struct WarpBuf {
    float d[CAP];                 // fp32 d2 of buffered candidates
    int32_t p[CAP];               // their sorted positions
    unsigned long long key[CAP];  // exact path: float64 d2 bits
    int32_t id[CAP];              // exact path: original ids
    int32_t cp[CAP];              // exact path: positions (payload)
    int32_t span_s[32];           // span compaction scratch
    int32_t span_l[32];
};

template <int NV>
struct QV {  // query coordinates passed by value (keeps them out of local memory)
    float v[4 * NV];
};

template <int NV>
__device__ __forceinline__ QV<NV> qv_of(const float (&q)[4 * NV]) {
    QV<NV> r;
#pragma unroll
    for (int i = 0; i < 4 * NV; ++i) r.v[i] = q[i];
    return r;
}

struct MT {  // (count, tau) result of a compaction
    int m;
    float tau;
};

struct Counters {
    int regions = 0, chunks = 0, appends = 0, compacts = 0, rows = 0, spec_fail = 0, exact = 0;
};

template <int NV, int DB>
struct Query {
    float q[4 * NV];
    int c[DB];      // cell per binned dim
    float qc[DB];   // position in cell units, (q - min) / width
    float w[DB];    // widths
    float invw[DB];
    int32_t p;
    int64_t cell_base;
};

__device__ __forceinline__ void store_d2(const KnnArgs& a, int64_t off, double v) {
    if (a.flags & FG_KNN_D2_F64)
        reinterpret_cast<double*>(a.out_d2)[off] = v;
    else
        reinterpret_cast<float*>(a.out_d2)[off] = (float)v;
}

template <int NV>
__device__ __forceinline__ float fp32_d2(const float (&q)[4 * NV], const float4* c) {
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const float4 x = c[j];
        float t;
        t = q[4 * j + 0] - x.x; acc = fmaf(t, t, acc);
        t = q[4 * j + 1] - x.y; acc = fmaf(t, t, acc);
        t = q[4 * j + 2] - x.z; acc = fmaf(t, t, acc);
        t = q[4 * j + 3] - x.w; acc = fmaf(t, t, acc);
    }
    return acc;
}

template <int NV>
__device__ __forceinline__ double exact_pos_d2(const KnnArgs& a, const float (&q)[4 * NV],
                                               int32_t cpos) {
    float c[4 * NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const float4 x = a.sc[(int64_t)cpos * NV + j];
        c[4 * j] = x.x; c[4 * j + 1] = x.y; c[4 * j + 2] = x.z; c[4 * j + 3] = x.w;
    }
    return exact_d2<4 * NV>(q, c, a.n_c);
}

// ---------------------------------------------------------------- exact path
// Bitonic sort of buf.(key,id,cp)[0..len) by (key, id); len is a power of 2.
template <int CAP>
__device__ void warp_sort_exact(WarpBuf<CAP>& b, int len) {
    const int lane = lane_id();
    for (int size = 2; size <= len; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const int sh = __ffs(stride) - 1;
            for (int i = lane; i < (len >> 1); i += 32) {
                const int x = ((i >> sh) << (sh + 1)) | (i & (stride - 1)), y = x + stride;
                const bool up = (x & size) == 0;
                const unsigned long long kx = b.key[x], ky = b.key[y];
                const int32_t ix = b.id[x], iy = b.id[y];
                const bool gt = kx > ky || (kx == ky && ix > iy);
                if (gt == up) {
                    b.key[x] = ky; b.key[y] = kx;
                    b.id[x] = iy; b.id[y] = ix;
                    const int32_t t = b.cp[x]; b.cp[x] = b.cp[y]; b.cp[y] = t;
                }
            }
            __syncwarp();
        }
    }
}

// Exact keys for buffer entries [0, m) (beyond-radius entries get the
// sentinel), sorted by (d2_f64, original index).
template <int NV, int CAP>
__device__ __noinline__ void exact_keys_and_sort(const KnnArgs& a, WarpBuf<CAP>& b, int m,
                                                 const QV<NV> qv) {
    const float(&q)[4 * NV] = qv.v;
    const int lane = lane_id();
    int len = 32;
    while (len < m) len <<= 1;
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    for (int e = lane; e < len; e += 32) {
        if (e < m) {
            const int32_t cpos = b.p[e];
            const double d = exact_pos_d2<NV>(a, q, cpos);
            const bool ok = !use_r2 || d <= a.max_r2;
            b.key[e] = ok ? (unsigned long long)__double_as_longlong(d) : ~0ull;
            b.id[e] = ok ? a.sid[cpos] : 0x7fffffff;
            b.cp[e] = cpos;
        } else {
            b.key[e] = ~0ull;
            b.id[e] = 0x7fffffff;
            b.cp[e] = -1;
        }
    }
    __syncwarp();
    warp_sort_exact<CAP>(b, len);
}

// ---------------------------------------------------------------- compaction
// Radix-select an upper bound T of the need-th smallest fp32 d2 on its top 16
// bits (only the bits where the smallest and largest prefix differ are
// searched), keep entries <= T*(1+1e-5); when that frees too little (massive
// ties) keep exactly the `need` best by exact key.  Returns the new count and
// tightens tau.
template <int NV, int CAP>
__device__ __noinline__ MT compact_impl(const KnnArgs& a, WarpBuf<CAP>& b, int m, int need,
                                       float tau, const QV<NV> q) {
    const int lane = lane_id();
    constexpr int PER = CAP / 32;
    unsigned pref[PER];
    float dv[PER];
    int32_t pv[PER];
    unsigned lo_p = 0xffffffffu, hi_p = 0u;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int e = i * 32 + lane;
        dv[i] = e < m ? b.d[e] : kInf;
        pv[i] = e < m ? b.p[e] : 0;
        pref[i] = __float_as_uint(dv[i]) >> 16;
        if (e < m) {
            lo_p = min(lo_p, pref[i]);
            hi_p = max(hi_p, pref[i]);
        }
    }
    lo_p = __reduce_min_sync(FG_FULL_MASK, lo_p);
    hi_p = __reduce_max_sync(FG_FULL_MASK, hi_p);
    const int nbits = 32 - __clz(lo_p ^ hi_p);
    unsigned P = nbits >= 32 ? 0u : (lo_p & ~((1u << nbits) - 1u));
#pragma unroll 1
    for (int bit = nbits - 1; bit >= 0; --bit) {
        const unsigned t = P | ((1u << bit) - 1u);
        int c = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) c += pref[i] <= t ? 1 : 0;
        c = __reduce_add_sync(FG_FULL_MASK, c);
        if (c < need) P |= 1u << bit;
    }
    const float T = __uint_as_float((P << 16) | 0xffffu);
    const float nt = fminf(tau, T * kMargin + kTiny);
    __syncwarp();
    int w = 0;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const bool keep = (i * 32 + lane) < m && dv[i] <= nt;
        const unsigned bal = __ballot_sync(FG_FULL_MASK, keep);
        if (keep) {
            const int pos = w + __popc(bal & lanemask_lt());
            b.d[pos] = dv[i];
            b.p[pos] = pv[i];
        }
        w += __popc(bal);
    }
    tau = nt;
    __syncwarp();
    if (w <= CAP - 32) return MT{w, tau};
    exact_keys_and_sort<NV, CAP>(a, b, w, q);
    int kept = 0;
    float mx = 0.0f;
    for (int base = 0; base < need; base += 32) {
        const int e = base + lane;
        const unsigned long long key = e < need ? b.key[e] : ~0ull;
        const bool ok = key != ~0ull;
        if (ok) {
            const float df = __double2float_ru(__longlong_as_double((long long)key));
            b.d[e] = df;
            b.p[e] = b.cp[e];
            mx = fmaxf(mx, df);
        }
        kept += __popc(__ballot_sync(FG_FULL_MASK, ok));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(FG_FULL_MASK, mx, o));
    if (kept >= need) tau = fminf(tau, mx * kMargin + kTiny);
    __syncwarp();
    return MT{kept, tau};
}

template <int NV, int CAP>
__device__ __forceinline__ int compact(const KnnArgs& a, WarpBuf<CAP>& b, int m, int need,
                                       float& tau, const float (&q)[4 * NV], Counters& cnt) {
    ++cnt.compacts;
    const MT r = compact_impl<NV, CAP>(a, b, m, need, tau, qv_of<NV>(q));
    tau = r.tau;
    return r.m;
}

// ---------------------------------------------------------------- geometry
// Smallest cube radius covering the tau-ball around q inside the grid.
template <int NV, int DB>
__device__ __forceinline__ int cover_radius(const Query<NV, DB>& Q, int nb, float tau) {
    const float rad = sqrtf(tau) * kMargin;
    int R = 0;
#pragma unroll
    for (int i = 0; i < DB; ++i) {
        const float rc = rad * Q.invw[i] + kCellSlack;
        const int lo = (int)fmaxf(floorf(Q.qc[i] - rc), -1.0f);
        const int hi = (int)fminf(floorf(Q.qc[i] + rc), (float)nb);
        R = max(R, max(min(Q.c[i], Q.c[i] - lo), min(nb - 1 - Q.c[i], hi - Q.c[i])));
    }
    return R;
}

template <int NV, int DB>
__device__ __forceinline__ int grid_radius(const Query<NV, DB>& Q, int nb) {
    int R = 0;
#pragma unroll
    for (int i = 0; i < DB; ++i) R = max(R, max(Q.c[i], nb - 1 - Q.c[i]));
    return R;
}

// Row r of a clipped lead box -> lead cells (last lead dim fastest).  Uses a
// float reciprocal: exact for the box sizes a grid of <= 30^4 rows can have.
template <int NL>
__device__ __forceinline__ void decode_row(int r, const int (&lo)[NL > 0 ? NL : 1],
                                           const int (&len)[NL > 0 ? NL : 1],
                                           const float (&inv)[NL > 0 ? NL : 1],
                                           int (&j)[NL > 0 ? NL : 1]) {
#pragma unroll
    for (int i = NL - 1; i >= 0; --i) {
        const int t = __float2int_rz(((float)r + 0.5f) * inv[i]);
        j[i] = lo[i] + (r - t * len[i]);
        r = t;
    }
}

// Expected squared distance of the need-th neighbour from the density of the
// 3^DB cube around the query's cell, inflated by kAlpha.  A hint only: the
// search certifies it (or restarts), so it never affects the answer.
template <int NV, int DB>
__device__ float density_tau(const KnnArgs& a, const Query<NV, DB>& Q, int need) {
    constexpr int NL = DB - 1;
    const int lane = lane_id();
    const int nb = a.nb;
    int lo_d[NL > 0 ? NL : 1], len_d[NL > 0 ? NL : 1];
    float inv[NL > 0 ? NL : 1];
    int rows = 1;
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        lo_d[i] = max(Q.c[i] - 1, 0);
        len_d[i] = min(Q.c[i] + 1, nb - 1) - lo_d[i] + 1;
        inv[i] = __frcp_rn((float)len_d[i]);
        rows *= len_d[i];
    }
    const int A = max(Q.c[NL] - 1, 0), B = min(Q.c[NL] + 1, nb - 1);
    int cnt = 0;
    for (int r = lane; r < rows; r += 32) {
        int jd[NL > 0 ? NL : 1];
        decode_row<NL>(r, lo_d, len_d, inv, jd);
        int rowflat = 0;
#pragma unroll
        for (int i = 0; i < NL; ++i) rowflat = rowflat * nb + jd[i];
        const int64_t rc = Q.cell_base + (int64_t)rowflat * nb;
        cnt += a.bounds[rc + B + 1] - a.bounds[rc + A];
    }
    cnt = __reduce_add_sync(FG_FULL_MASK, cnt);
    if (cnt < 2 * need + 2) return kInf;  // too sparse to trust
    float vol = (float)(rows * (B - A + 1));
#pragma unroll
    for (int i = 0; i < DB; ++i) vol *= Q.w[i];
    constexpr float vd = DB == 1 ? 2.0f : DB == 2 ? 3.14159265f : DB == 3 ? 4.18879020f
                       : DB == 4 ? 4.93480220f : 5.26378901f;  // unit-ball volume
    const float x = (float)need * vol / ((float)cnt * vd);
    const float rho = exp2f(__log2f(x) * (1.0f / (float)DB));
    return (kAlpha * rho) * (kAlpha * rho);
}

struct Filter {
    bool use_dir, use_r2;
    float r2_lo, r2_hi;
};

// Evaluate one group of spans (one per lane: start S, length L) and append
// the passing candidates.
template <int NV, int DB, int CAP, bool FILT>
__device__ __forceinline__ void scan_spans(const KnnArgs& a, WarpBuf<CAP>& b,
                                           const Query<NV, DB>& Q, int32_t S, int32_t L, int& m,
                                           int need, float& tau, const Filter& flt, Counters& cnt) {
    const int lane = lane_id();
    const unsigned nonempty = __ballot_sync(FG_FULL_MASK, L > 0);
    if (!nonempty) return;
    // Short spans (uniform data: a trimmed row holds a few points): every lane
    // walks its own span; the warp runs max(L) steps with no flattening.  Long
    // spans (clusters): flatten into full 32-candidate chunks below.
    const int max_len = __reduce_max_sync(FG_FULL_MASK, (unsigned)L);
    const int total = __reduce_add_sync(FG_FULL_MASK, (unsigned)L);
    if (FG_SPAN_WALK && max_len * 2 <= ((total + 31) >> 5) * 5) {
        for (int i = 0; i < max_len; ++i) {
            ++cnt.chunks;
            const bool live = i < L;
            const int32_t cpos = S + i;
            bool pass = false;
            float d2 = kInf;
            if (live) {
                d2 = fp32_d2<NV>(Q.q, a.sc + (int64_t)cpos * NV);
                pass = d2 <= tau && cpos != Q.p;
            }
            if (FILT && flt.use_dir && pass) {
                const int8_t role = a.dir[a.sid[cpos]];
                pass = role == 0 || role == 3;
            }
            if (FILT && flt.use_r2 && pass) {
                if (d2 > flt.r2_hi)
                    pass = false;
                else if (d2 >= flt.r2_lo)
                    pass = exact_pos_d2<NV>(a, Q.q, cpos) <= a.max_r2;
            }
            unsigned bal = __ballot_sync(FG_FULL_MASK, pass);
            if (bal) {
                if (m + __popc(bal) > CAP) {
                    m = compact<NV, CAP>(a, b, m, need, tau, Q.q, cnt);
                    pass = pass && d2 <= tau;
                    bal = __ballot_sync(FG_FULL_MASK, pass);
                }
                if (pass) {
                    const int pos = m + __popc(bal & lanemask_lt());
                    b.d[pos] = d2;
                    b.p[pos] = cpos;
                }
                m += __popc(bal);
                cnt.appends += __popc(bal);
                __syncwarp();
            }
        }
        return;
    }
    const int ns = __popc(nonempty);
    if (L > 0) {
        const int dst = __popc(nonempty & lanemask_lt());
        b.span_s[dst] = S;
        b.span_l[dst] = L;
    }
    __syncwarp();
    S = lane < ns ? b.span_s[lane] : 0;
    L = lane < ns ? b.span_l[lane] : 0;
    __syncwarp();
    const int32_t incl = warp_inclusive_scan(L);
    const int32_t excl = incl - L;
    const int32_t T = __shfl_sync(FG_FULL_MASK, incl, 31);
    const unsigned le = (2u << lane) - 1u;
    for (int32_t f0 = 0; f0 < T; f0 += 32) {
        ++cnt.chunks;
        const int base = __popc(__ballot_sync(FG_FULL_MASK, lane < ns && incl <= f0));
        const unsigned starts = __reduce_or_sync(
            FG_FULL_MASK, (lane < ns && excl > f0 && excl < f0 + 32) ? 1u << (excl - f0) : 0u);
        const int sidx = min(base + __popc(starts & le), 31);
        const int32_t Ss = __shfl_sync(FG_FULL_MASK, S, sidx);
        const int32_t Es = __shfl_sync(FG_FULL_MASK, excl, sidx);
        const int32_t f = f0 + lane;
        const int32_t cpos = Ss + (f - Es);
        bool pass = false;
        float d2 = kInf;
        if (f < T) {
            d2 = fp32_d2<NV>(Q.q, a.sc + (int64_t)cpos * NV);
            pass = d2 <= tau && cpos != Q.p;
        }
        if (FILT && flt.use_dir && pass) {
            const int8_t role = a.dir[a.sid[cpos]];
            pass = role == 0 || role == 3;
        }
        if (FILT && flt.use_r2 && pass) {
            if (d2 > flt.r2_hi)
                pass = false;
            else if (d2 >= flt.r2_lo)
                pass = exact_pos_d2<NV>(a, Q.q, cpos) <= a.max_r2;
        }
        unsigned bal = __ballot_sync(FG_FULL_MASK, pass);
        if (bal) {
            if (m + __popc(bal) > CAP) {
                m = compact<NV, CAP>(a, b, m, need, tau, Q.q, cnt);
                pass = pass && d2 <= tau;
                bal = __ballot_sync(FG_FULL_MASK, pass);
            }
            if (pass) {
                const int pos = m + __popc(bal & lanemask_lt());
                b.d[pos] = d2;
                b.p[pos] = cpos;
            }
            m += __popc(bal);
            cnt.appends += __popc(bal);
            __syncwarp();
        }
    }
}

// Scan region (R_old, R_new]; R_old = -1 means the whole cube(R_new).
template <int NV, int DB, int CAP, bool FILT>
__device__ void scan_region(const KnnArgs& a, WarpBuf<CAP>& b, const Query<NV, DB>& Q, int R_old,
                            int R_new, bool prune, int& m, int need, float& tau, const Filter& flt,
                            Counters& cnt) {
    constexpr int NL = DB - 1;
    const int lane = lane_id();
    const int nb = a.nb;
    int lo_d[NL > 0 ? NL : 1], len_d[NL > 0 ? NL : 1];
    float inv[NL > 0 ? NL : 1];
    int rows = 1;
#pragma unroll
    for (int i = 0; i < NL; ++i) {
        lo_d[i] = max(Q.c[i] - R_new, 0);
        len_d[i] = min(Q.c[i] + R_new, nb - 1) - lo_d[i] + 1;
        inv[i] = __frcp_rn((float)len_d[i]);
        rows *= len_d[i];
    }
    ++cnt.regions;
    cnt.rows += rows;
    const int cl = Q.c[NL];
    const float qcl = Q.qc[NL];
    const int A = max(cl - R_new, 0), B = min(cl + R_new, nb - 1);
    for (int rb = 0; rb < rows; rb += 32) {
        const int r = rb + lane;
        int32_t S0 = 0, L0 = 0, S1 = 0, L1 = 0;
        if (r < rows) {
            int jd[NL > 0 ? NL : 1];
            decode_row<NL>(r, lo_d, len_d, inv, jd);
            int maxabs = 0, rowflat = 0;
            float bd2 = 0.0f;
#pragma unroll
            for (int i = 0; i < NL; ++i) {
                rowflat = rowflat * nb + jd[i];
                maxabs = max(maxabs, abs(jd[i] - Q.c[i]));
                const float fj = (float)jd[i];
                float g = fmaxf(fmaxf(fj - Q.qc[i], Q.qc[i] - (fj + 1.0f)) - kCellSlack, 0.0f);
                g *= Q.w[i];
                bd2 = fmaf(g, g, bd2);
            }
            int a0 = A, b0 = B, a1 = 1, b1 = 0;
            if (maxabs <= R_old) {
                b0 = cl - R_old - 1;
                a1 = cl + R_old + 1;
                b1 = B;
            }
            if (prune) {
                const float rem = tau - bd2;
                const float rc = sqrtf(fmaxf(rem, 0.0f)) * Q.invw[NL] * kMargin + kCellSlack;
                const int wa = (int)fmaxf(floorf(qcl - rc), -1.0f);
                const int wb = rem < 0.0f ? -2 : (int)fminf(floorf(qcl + rc), (float)nb);
                a0 = max(a0, wa); b0 = min(b0, wb);
                a1 = max(a1, wa); b1 = min(b1, wb);
            }
            const int64_t rowcell = Q.cell_base + (int64_t)rowflat * nb;
            if (a0 <= b0) {
                S0 = a.bounds[rowcell + a0];
                L0 = a.bounds[rowcell + b0 + 1] - S0;
            }
            if (a1 <= b1) {
                S1 = a.bounds[rowcell + a1];
                L1 = a.bounds[rowcell + b1 + 1] - S1;
            }
        }
        scan_spans<NV, DB, CAP, FILT>(a, b, Q, S0, L0, m, need, tau, flt, cnt);
        if (R_old >= 0) scan_spans<NV, DB, CAP, FILT>(a, b, Q, S1, L1, m, need, tau, flt, cnt);
    }
}

template <int NV, int DB, int CAP>
__device__ __forceinline__ void scan(const KnnArgs& a, WarpBuf<CAP>& b, const Query<NV, DB>& Q,
                                     int R_old, int R_new, bool prune, int& m, int need, float& tau,
                                     const Filter& flt, Counters& cnt) {
    if (flt.use_dir || flt.use_r2)
        scan_region<NV, DB, CAP, true>(a, b, Q, R_old, R_new, prune, m, need, tau, flt, cnt);
    else
        scan_region<NV, DB, CAP, false>(a, b, Q, R_old, R_new, prune, m, need, tau, flt, cnt);
}

// ---------------------------------------------------------------- epilogue
// Fast path for m <= 64: key = float32(d2_f64) bits (monotone for d2 >= 0),
// lane l owns entries l and l+32; every entry's output slot is its rank, i.e.
// the number of entries with a smaller key (counted against keys broadcast
// from shared memory).  If two valid entries share a key and one of them
// lands in the row (rank < need), the float32 keys cannot decide the order
// (exact ties / sub-ulp near-ties): returns false and the exact path runs.
template <int NV, int CAP>
__device__ bool epilogue_fast(const KnnArgs& a, WarpBuf<CAP>& b, const float (&q)[4 * NV], int m,
                              int need, int64_t row_out) {
    const int lane = lane_id();
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    unsigned key[2];
    int32_t pos[2];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int e = lane + 32 * t;
        key[t] = ~0u;
        pos[t] = -1;
        if (e < m) {
            pos[t] = b.p[e];
            const double d = exact_pos_d2<NV>(a, q, pos[t]);
            if (!use_r2 || d <= a.max_r2) key[t] = __float_as_uint(__double2float_rn(d));
        }
    }
    unsigned* kb = reinterpret_cast<unsigned*>(b.key);  // reuse as a 32-bit key array
    __syncwarp();
    kb[lane] = key[0];
    kb[lane + 32] = key[1];
    __syncwarp();
    int rank[2] = {0, 0}, same[2] = {0, 0};
    for (int j = 0; j < m; ++j) {
        const unsigned kj = kb[j];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            rank[t] += kj < key[t] ? 1 : 0;
            same[t] += kj == key[t] ? 1 : 0;
        }
    }
    bool amb = false;
#pragma unroll
    for (int t = 0; t < 2; ++t) amb |= key[t] != ~0u && same[t] > 1 && rank[t] < need;
    if (__any_sync(FG_FULL_MASK, amb)) return false;
    const bool f64 = a.flags & FG_KNN_D2_F64;
    int valid = 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        valid += key[t] != ~0u ? 1 : 0;
        if (key[t] != ~0u && rank[t] < need) {
            const int64_t off = row_out + 1 + rank[t];
            a.out_idx[off] = a.sid[pos[t]];
            if (f64)
                reinterpret_cast<double*>(a.out_d2)[off] = exact_pos_d2<NV>(a, q, pos[t]);
            else
                reinterpret_cast<float*>(a.out_d2)[off] = __uint_as_float(key[t]);
        }
    }
    valid = __reduce_add_sync(FG_FULL_MASK, valid);
    for (int sl = valid + lane; sl < need; sl += 32) {  // padding
        a.out_idx[row_out + 1 + sl] = -1;
        store_d2(a, row_out + 1 + sl, 0.0);
    }
    return true;
}

// Alternative fast path: register bitonic sort of (float32(d2_f64), position),
// E keys per lane (FG_EPI_BITONIC).
template <int NV, int E, int CAP>
__device__ bool epilogue_bitonic(const KnnArgs& a, WarpBuf<CAP>& b, const float (&q)[4 * NV], int m,
                              int need, int64_t row_out) {
    constexpr int N = 32 * E;
    const int lane = lane_id();
    const bool use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    unsigned kx[E];  // float32(d2_f64) bits (monotone for d2 >= 0); invalid = ~0
    int32_t px[E];   // sorted position
#pragma unroll
    for (int t = 0; t < E; ++t) {
        const int e = E * lane + t;
        kx[t] = ~0u;
        px[t] = -1;
        if (e < m) {
            const int32_t cpos = b.p[e];
            const double d = exact_pos_d2<NV>(a, q, cpos);
            if (!use_r2 || d <= a.max_r2) {
                kx[t] = __float_as_uint(__double2float_rn(d));
                px[t] = cpos;
            }
        }
    }
#pragma unroll
    for (int k2 = 2; k2 <= N; k2 <<= 1) {
#pragma unroll
        for (int j2 = k2 >> 1; j2 > 0; j2 >>= 1) {
            if (j2 < E) {
#pragma unroll
                for (int t = 0; t < E; ++t) {
                    if ((t & j2) == 0) {
                        const int u = t | j2;
                        const bool asc = ((E * lane + t) & k2) == 0;
                        const bool sw = asc ? (kx[t] > kx[u]) : (kx[t] < kx[u]);
                        const unsigned k0 = sw ? kx[u] : kx[t], k1 = sw ? kx[t] : kx[u];
                        const int32_t p0 = sw ? px[u] : px[t], p1 = sw ? px[t] : px[u];
                        kx[t] = k0; kx[u] = k1; px[t] = p0; px[u] = p1;
                    }
                }
            } else {
#pragma unroll
                for (int t = 0; t < E; ++t) {
                    const int i = E * lane + t;
                    const unsigned ok = __shfl_xor_sync(FG_FULL_MASK, kx[t], j2 / E);
                    const int32_t op = __shfl_xor_sync(FG_FULL_MASK, px[t], j2 / E);
                    const bool keep_min = ((i & j2) == 0) == ((i & k2) == 0);
                    const bool take = keep_min ? (ok < kx[t]) : (ok > kx[t]);
                    kx[t] = take ? ok : kx[t];
                    px[t] = take ? op : px[t];
                }
            }
        }
    }
    // entries that decide the row: pairs (i, i+1) with i + 1 <= need
    bool amb = false;
#pragma unroll
    for (int t = 0; t + 1 < E; ++t) {
        const int i = E * lane + t;
        amb |= i + 1 <= need && kx[t + 1] != ~0u && kx[t] == kx[t + 1];
    }
    {
        const unsigned nxt = __shfl_down_sync(FG_FULL_MASK, kx[0], 1);
        const int i = E * lane + E - 1;
        amb |= lane < 31 && i + 1 <= need && nxt != ~0u && kx[E - 1] == nxt;
    }
    if (__any_sync(FG_FULL_MASK, amb)) return false;
    const bool f64 = a.flags & FG_KNN_D2_F64;
#pragma unroll
    for (int t = 0; t < E; ++t) {
        const int i = E * lane + t;
        if (i < need) {
            const int64_t off = row_out + 1 + i;
            if (kx[t] != ~0u) {
                a.out_idx[off] = a.sid[px[t]];
                if (f64)
                    reinterpret_cast<double*>(a.out_d2)[off] = exact_pos_d2<NV>(a, q, px[t]);
                else
                    reinterpret_cast<float*>(a.out_d2)[off] = __uint_as_float(kx[t]);
            } else {
                a.out_idx[off] = -1;
                store_d2(a, off, 0.0);
            }
        }
    }
    return true;
}

template <int NV, int CAP>
__device__ __noinline__ void epilogue_exact(const KnnArgs& a, WarpBuf<CAP>& b, const QV<NV> q, int m,
                                            int k, int64_t row_out) {
    const int lane = lane_id();
    exact_keys_and_sort<NV, CAP>(a, b, m, q);
    for (int sl = 1 + lane; sl < k; sl += 32) {
        const int e = sl - 1;
        const unsigned long long key = e < m ? b.key[e] : ~0ull;
        if (key != ~0ull) {
            a.out_idx[row_out + sl] = b.id[e];
            store_d2(a, row_out + sl, __longlong_as_double((long long)key));
        } else {
            a.out_idx[row_out + sl] = -1;
            store_d2(a, row_out + sl, 0.0);
        }
    }
}

// ---------------------------------------------------------------- per-query pieces
template <int NV, int DB>
__device__ __forceinline__ void setup_query(const KnnArgs& a, int64_t p, Query<NV, DB>& Q) {
    const int nb = a.nb;
    Q.p = (int32_t)p;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const float4 x = a.sc[p * NV + j];
        Q.q[4 * j] = x.x; Q.q[4 * j + 1] = x.y; Q.q[4 * j + 2] = x.z; Q.q[4 * j + 3] = x.w;
    }
    const int s = a.n_splits == 1 ? 0 : split_of(a.rs, a.n_splits, p);
    Q.cell_base = (int64_t)s * a.total;
#pragma unroll
    for (int i = 0; i < DB; ++i) {
        const float mn = (float)a.mins[(int64_t)s * DB + i];  // a float32 value
        Q.w[i] = (float)a.widths[(int64_t)s * DB + i];
        Q.invw[i] = __frcp_rn(Q.w[i]);
        Q.qc[i] = (Q.q[i] - mn) * Q.invw[i];
        Q.c[i] = min(max(__float2int_rd(Q.qc[i]), 0), nb - 1);
    }
}

// Self slot; padding of a row that runs no query.  Returns true when the
// query is skipped (k == 1, or its role is 0/2).
__device__ __forceinline__ bool begin_row(const KnnArgs& a, int32_t qid, int64_t row_out, int need,
                                          const Filter& flt) {
    const int lane = lane_id();
    if (lane == 0) {
        a.out_idx[row_out] = qid;
        store_d2(a, row_out, 0.0);
    }
    const bool skip = need == 0 || (flt.use_dir && (a.dir[qid] == 0 || a.dir[qid] == 2));
    if (skip) {
        for (int s = 1 + lane; s < a.k; s += 32) {
            a.out_idx[row_out + s] = -1;
            store_d2(a, row_out + s, 0.0);
        }
    }
    return skip;
}

// Plain growth from the query's own cell (or its 3^d cube): regions until the
// cover radius of tau is scanned.  Fills buf.  Out of line (rare path), so
// everything crosses by value: nothing of the hot path becomes address-taken.
struct PlainOut {
    int m;
    float tau;
    Counters cnt;
};

template <int NV, int DB, int CAP>
__device__ __noinline__ PlainOut plain_search(const KnnArgs& a, WarpBuf<CAP>& buf,
                                              const Query<NV, DB> Q, int32_t qid, int need,
                                              const Filter flt, float tau) {
    Counters cnt;
    const int nb = a.nb;
    const int R_grid = grid_radius(Q, nb);
    int m = 0, R_done = -1;
    const int64_t own = a.bin_idx[qid];
    const int own_cnt = a.bounds[own + 1] - a.bounds[own];
    int R_next = own_cnt > need ? 0 : min(1, R_grid);
    while (R_next > R_done) {
        scan<NV, DB, CAP>(a, buf, Q, R_done, R_next, tau < kInf, m, need, tau, flt, cnt);
        R_done = R_next;
        if (R_done >= R_grid) break;
        if (m >= need) m = compact<NV, CAP>(a, buf, m, need, tau, Q.q, cnt);
        R_next = tau < kInf ? cover_radius(Q, nb, tau) : R_done + 1;
    }
    return PlainOut{m, tau, cnt};
}

__device__ __forceinline__ void add_counters(Counters& c, const Counters& d) {
    c.regions += d.regions;
    c.chunks += d.chunks;
    c.appends += d.appends;
    c.compacts += d.compacts;
    c.rows += d.rows;
    c.spec_fail += d.spec_fail;
    c.exact += d.exact;
}

// >= need buffered entries strictly inside tau0 (3e-5 margin): certified.
template <int CAP>
__device__ __forceinline__ bool certified(const WarpBuf<CAP>& buf, int m, int need, float tau0) {
    const float inner = tau0 * (1.0f - 3e-5f);
    int c_in = 0;
    for (int e = lane_id(); e < m; e += 32) c_in += buf.d[e] <= inner ? 1 : 0;
    return __reduce_add_sync(FG_FULL_MASK, c_in) >= need;
}

template <int NV, int CAP>
__device__ __forceinline__ void finish_query(const KnnArgs& a, WarpBuf<CAP>& buf,
                                             const float (&q)[4 * NV], int m, int need, float tau,
                                             int64_t row_out, Counters& cnt) {
    bool done = false;
    if (m > FG_EPI_CUT && need <= 63) m = compact<NV, CAP>(a, buf, m, need, tau, q, cnt);
#if FG_EPI_BITONIC
    if (m <= 64 && need <= 63) done = epilogue_bitonic<NV, 2, CAP>(a, buf, q, m, need, row_out);
#else
    if (m <= 64 && need <= 63) done = epilogue_fast<NV, CAP>(a, buf, q, m, need, row_out);
#endif
    if (!done) {
        ++cnt.exact;
        epilogue_exact<NV, CAP>(a, buf, qv_of<NV>(q), m, a.k, row_out);
    }
    __syncwarp();
}

__device__ __forceinline__ Filter make_filter(const KnnArgs& a) {
    Filter flt;
    flt.use_dir = a.flags & FG_KNN_USE_DIRECTION;
    flt.use_r2 = a.flags & FG_KNN_USE_MAX_R2;
    flt.r2_hi = flt.use_r2 ? (float)(a.max_r2 * (1.0 + 1e-5)) + kTiny : 0.0f;
    flt.r2_lo = flt.use_r2 ? (float)(a.max_r2 * (1.0 - 1e-5)) : 0.0f;
    return flt;
}

__device__ __forceinline__ void flush_stats(const KnnArgs& a, int64_t queries, const Counters& cnt) {
    if (a.stats && lane_id() == 0) {
        atomicAdd(&a.stats[ST_QUERIES], (unsigned long long)queries);
        atomicAdd(&a.stats[ST_REGIONS], (unsigned long long)cnt.regions);
        atomicAdd(&a.stats[ST_CHUNKS], (unsigned long long)cnt.chunks);
        atomicAdd(&a.stats[ST_APPENDS], (unsigned long long)cnt.appends);
        atomicAdd(&a.stats[ST_COMPACT], (unsigned long long)cnt.compacts);
        atomicAdd(&a.stats[ST_SPEC_FAIL], (unsigned long long)cnt.spec_fail);
        atomicAdd(&a.stats[ST_EXACT_EPI], (unsigned long long)cnt.exact);
        atomicAdd(&a.stats[ST_ROWS], (unsigned long long)cnt.rows);
    }
}

// ---------------------------------------------------------------- kernel (one query per warp)
template <int NV, int DB, int CAP>
__global__ void __launch_bounds__(kWarpsPerBlock * 32, FG_KNN_MINB) k_knn_fwd(const __grid_constant__ KnnArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    WarpBuf<CAP>& buf = reinterpret_cast<WarpBuf<CAP>*>(smem_raw)[threadIdx.x >> 5];
    const int64_t warp_global = blockIdx.x * (int64_t)kWarpsPerBlock + (threadIdx.x >> 5);
    const int64_t warps_total = (int64_t)gridDim.x * kWarpsPerBlock;
    const int need = a.k - 1;
    const Filter flt = make_filter(a);
    const float r2_tau = flt.use_r2 ? flt.r2_hi : kInf;
    const bool exhaustive = a.flags & FG_KNN_EXHAUSTIVE;
    Counters cnt;
    int64_t queries = 0;
    const bool use_list = a.qlist && !(a.qall && (int64_t)*a.qall * 4 > a.n);
    const int64_t n_q = use_list ? (int64_t)*a.qcount : a.n;
    for (int64_t i = warp_global; i < n_q; i += warps_total) {
        const int64_t p = use_list ? (int64_t)a.qlist[i] : i;
        ++queries;
        const int32_t qid = a.sid[p];
        const int64_t row_out = (int64_t)qid * a.k;
        if (begin_row(a, qid, row_out, need, flt)) continue;
        Query<NV, DB> Q;
        setup_query(a, p, Q);
        float tau = r2_tau;
        int m = 0;
        if (exhaustive) {
            scan<NV, DB, CAP>(a, buf, Q, -1, grid_radius(Q, a.nb), false, m, need, tau, flt, cnt);
        } else {
            bool done = false;
            const float tau0 = a.n_c == DB ? density_tau(a, Q, need) : kInf;
            if (tau0 < tau) {
                float t0 = tau0;
                const int R0 = cover_radius(Q, a.nb, tau0);
                scan<NV, DB, CAP>(a, buf, Q, -1, R0, true, m, need, t0, flt, cnt);
                if (certified(buf, m, need, tau0)) {
                    tau = t0;
                    done = true;
                } else {
                    ++cnt.spec_fail;
                }
            }
            if (!done) {
                const PlainOut po = plain_search<NV, DB, CAP>(a, buf, Q, qid, need, flt, tau);
                m = po.m;
                tau = po.tau;
                add_counters(cnt, po.cnt);
            }
        }
        finish_query<NV, CAP>(a, buf, Q.q, m, need, tau, row_out, cnt);
    }
    flush_stats(a, queries, cnt);
}

template <int NV, int DB, int CAP>
int launch_knn(const KnnArgs& a, cudaStream_t st) {
    const size_t smem = sizeof(WarpBuf<CAP>) * kWarpsPerBlock;
    auto kern = k_knn_fwd<NV, DB, CAP>;
    if (smem > 48 * 1024)
        FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int64_t blocks = std::min<int64_t>(ceil_div(a.n, kWarpsPerBlock),
                                             a.qlist ? (int64_t)148 * 64 : (int64_t)1 << 30);
    kern<<<(unsigned)blocks, kWarpsPerBlock * 32, smem, st>>>(a);
    return launched(st);
}

template <int NV, int DB>
int dispatch_cap(const KnnArgs& a, cudaStream_t st) {
    const int need = a.k - 1;
    if (need + 64 <= 128) return launch_knn<NV, DB, 128>(a, st);
    return launch_knn<NV, DB, 1024>(a, st);
}

// d_bin dispatch for one coordinate width (instantiated per NV in its own
// translation unit so the kernels compile in parallel).
template <int NV>
int dispatch_db(const KnnArgs& a, int d_bin, cudaStream_t st) {
    switch (d_bin) {
        case 1: return dispatch_cap<NV, 1>(a, st);
        case 2: return dispatch_cap<NV, 2>(a, st);
        case 3: return dispatch_cap<NV, 3>(a, st);
        case 4: return dispatch_cap<NV, 4>(a, st);
        default:
            if constexpr (NV >= 2) return dispatch_cap<NV, 5>(a, st);
            return FG_ERR_TOO_FEW_DIMS;
    }
}

int dispatch_nv1(const KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_nv2(const KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_nv3(const KnnArgs& a, int d_bin, cudaStream_t st);
int dispatch_nv4(const KnnArgs& a, int d_bin, cudaStream_t st);

}  // namespace search
}  // namespace fg
