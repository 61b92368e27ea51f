// fg_grad.cu -- binned_select_knn backward (replaces G/knn.py:135-168) for
// sm_100a.
//
// For every valid non-self slot (v, s) -> u with upstream g, the reference adds
// 2g(x_v - x_u) to grad[v] and its negation to grad[u] (np.add.at, fixed order:
// G/knn.py:160-167, bitwise repeatable, pkg/tests/test_knn.py:302-309).  Every
// term is formed exactly in float64 (fp32 g and x: a 24-bit by 25-bit product).
//
// FG_BWD_DETERMINISTIC ("transposed", namespace bt): bitwise repeatable, no
// floating-point atomics.
//   K7a k_bt_count    in-degree of every 512-position destination bucket (sorted
//                     order), shared-memory histograms, one global add per
//                     (CTA, bucket);
//   K7b k_scan        bucket offsets (the binning's look-back scan);
//   K7c k_bt_scatter  warp per row in sorted order: the query side of the row
//                     (float64 butterfly, fixed order) and one 8-byte entry
//                     (src id | dst position, g) per neighbour slot, staged in
//                     shared memory and written bucket-contiguously;
//   K7d k_bt_reduce   CTA per bucket: counting sort of its entries by
//                     destination in shared memory, then thread per
//                     destination sums its terms as int64 fixed point on a
//                     per-bucket quantum (integer addition is associative, so
//                     the result does not depend on the order entries arrived
//                     in), adds the query side and rounds once.
// Precision: a destination with m terms is exact to m * E * 2^-62 of the
// bucket's largest term (E = entries in the bucket; ~2^-42 at north_star),
// the query side to float64 rounding of its sum.
//
// Default (namespace grad): compensated fp32x4 atomics, float64-class accuracy,
// not bitwise repeatable.  Measured at north_star (1M x 40, B200): default
// 0.83 ms, transposed 1.36 ms -- the scattered-atomic path is bound by L2
// atomic throughput (~193 G ops/s for any RED width), the transposed one by
// the instruction and latency cost of its two counting sorts.
#include "fg_common.cuh"
#include "fg_scan.cuh"

#include <algorithm>

namespace fg {
namespace grad {

constexpr int kRowWarps = 8;

// Exact-to-~2^-48 accumulation with fp32x4 atomics: a float64 value x is
// split into hi = fp32(x) and lo = fp32(x - hi); hi is added with a returning
// vector atomic, the exact rounding error of that addition (TwoSum against the
// returned old value) plus lo is added to a second accumulator.  Two 16-byte
// L2 operations per 4 coordinates instead of four float64 atomics.
__device__ __forceinline__ void two_sum_add(float4* hi_acc, float4* lo_acc, const double (&x)[4]) {
    float4 h, l;
    float* hp = &h.x;
    float* lp = &l.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        hp[i] = (float)x[i];
        lp[i] = isfinite(x[i]) ? (float)(x[i] - (double)hp[i]) : 0.f;
    }
    const float4 old = atomicAdd(hi_acc, h);
    const float* op = &old.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float a = op[i], b = hp[i];
        const float sum = __fadd_rn(a, b);
        const float bb = __fsub_rn(sum, a);
        const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(sum, bb)), __fsub_rn(b, bb));
        // non-finite hi: the error terms are meaningless (inf - inf); hi carries the result
        lp[i] = isfinite(sum) ? __fadd_rn(lp[i], err) : 0.f;
    }
    atomicAdd(lo_acc, l);
}

// Warp per row (visited in `order` when given: spatially sorted rows keep the
// neighbour gathers and the atomic targets local), lanes over slots.
template <int NV, typename TC, typename TG>
__global__ void __launch_bounds__(kRowWarps * 32) k_knn_bwd(const TC* __restrict__ coords, int64_t n,
                                                          int n_c, const int32_t* __restrict__ idx,
                                                          int k, const TG* __restrict__ gd2,
                                                          const int32_t* __restrict__ order,
                                                          float4* __restrict__ hi,
                                                          float4* __restrict__ lo) {
    constexpr int NC = 4 * NV;
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= n) return;
    const int64_t v = order ? order[p] : p;
    double xv[NC], qs[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        xv[i] = i < n_c ? (double)coords[v * n_c + i] : 0.0;
        qs[i] = 0.0;
    }
    for (int base = 1; base < k; base += 32) {
        const int s = base + lane;
        const int32_t u = s < k ? idx[v * k + s] : -1;
        if (u >= 0) {
            const double two_g = 2.0 * (double)gd2[v * k + s];
#pragma unroll
            for (int j = 0; j < NV; ++j) {
                double c[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = 4 * j + e;
                    const double xu = i < n_c ? (double)coords[(int64_t)u * n_c + i] : 0.0;
                    // float32 inputs: exact (24-bit g times a 25-bit difference);
                    // float64 inputs: numpy's (2g) * (x_v - x_u), G/knn.py:164-165
                    c[e] = two_g * (xv[i] - xu);
                    qs[i] += c[e];
                    c[e] = -c[e];
                }
                two_sum_add(hi + (int64_t)u * NV + j, lo + (int64_t)u * NV + j, c);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < NC; ++i) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qs[i] += __shfl_xor_sync(FG_FULL_MASK, qs[i], o);
    }
    if (lane == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double c[4] = {qs[4 * j], qs[4 * j + 1], qs[4 * j + 2], qs[4 * j + 3]};
            two_sum_add(hi + v * NV + j, lo + v * NV + j, c);
        }
    }
}

// d == 4 with 16-byte aligned coordinates (the caller checks), k <= 65: RPW rows per warp with every (row, slot-round) chain in
// flight at once -- the coordinate gathers, then the returning fp32x4 atomics,
// then the TwoSum corrections -- so the L2 round trips of 2*RPW chains overlap
// (the warp-per-row kernel above waits for each one).  Same arithmetic.
template <int RPW, int SR>
__global__ void __launch_bounds__(kRowWarps * 32, 4) k_knn_bwd_pipe(
    const float* __restrict__ coords, int64_t n, int n_c, const int32_t* __restrict__ idx, int k,
    const float* __restrict__ gd2, const int32_t* __restrict__ order, float4* __restrict__ hi,
    float4* __restrict__ lo) {
    constexpr int C = RPW * SR;
    const int lane = lane_id();
    const int64_t p0 = (blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5)) * RPW;
    if (p0 >= n) return;
    int64_t v[RPW];
    int32_t u[C];
    float g[C];
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        const int64_t pr = min(p0 + r, n - 1);
        v[r] = order ? (int64_t)order[pr] : pr;
    }
#pragma unroll
    for (int r = 0; r < RPW; ++r)
#pragma unroll
        for (int q = 0; q < SR; ++q) {
            const int s = 1 + lane + 32 * q;
            const bool ok = p0 + r < n && s < k;
            u[r * SR + q] = ok ? idx[v[r] * k + s] : -1;
            g[r * SR + q] = ok ? gd2[v[r] * k + s] : 0.0f;
        }
    auto load4 = [&](int64_t w) {
        if (n_c == 4) return reinterpret_cast<const float4*>(coords)[w];
        float t[4] = {0.f, 0.f, 0.f, 0.f};
        for (int i = 0; i < n_c; ++i) t[i] = coords[w * n_c + i];
        return make_float4(t[0], t[1], t[2], t[3]);
    };
    float4 xv[RPW], xu[C];
#pragma unroll
    for (int r = 0; r < RPW; ++r) xv[r] = load4(v[r]);
#pragma unroll
    for (int c = 0; c < C; ++c) xu[c] = u[c] >= 0 ? load4(u[c]) : xv[c / SR];
    // returning hi atomics for every chain, then the corrections
    float4 h[C], old[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        const double tg = 2.0 * (double)g[c];
        const float4 a = xv[c / SR], b = xu[c];
        h[c] = make_float4((float)-(tg * ((double)a.x - (double)b.x)), (float)-(tg * ((double)a.y - (double)b.y)),
                           (float)-(tg * ((double)a.z - (double)b.z)), (float)-(tg * ((double)a.w - (double)b.w)));
        if (u[c] >= 0) old[c] = atomicAdd(hi + u[c], h[c]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if (u[c] < 0) continue;
        const double tg = 2.0 * (double)g[c];
        const float4 a = xv[c / SR], b = xu[c];
        const double x[4] = {-(tg * ((double)a.x - (double)b.x)), -(tg * ((double)a.y - (double)b.y)),
                             -(tg * ((double)a.z - (double)b.z)), -(tg * ((double)a.w - (double)b.w))};
        const float* hp = &h[c].x;
        const float* op = &old[c].x;
        float4 l;
        float* lp = &l.x;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            lp[i] = (float)(x[i] - (double)hp[i]);
            const float a2 = op[i], b2 = hp[i];
            const float sum = __fadd_rn(a2, b2);
            const float bb = __fsub_rn(sum, a2);
            const float err = __fadd_rn(__fsub_rn(a2, __fsub_rn(sum, bb)), __fsub_rn(b2, bb));
            lp[i] = isfinite(sum) ? __fadd_rn(lp[i], err) : 0.f;
        }
        atomicAdd(lo + u[c], l);
    }
    // query side: per row, the sum of its terms (float64 warp reduction)
#pragma unroll
    for (int r = 0; r < RPW; ++r) {
        double qs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < SR; ++q) {
            const int c = r * SR + q;
            if (u[c] < 0) continue;
            const double tg = 2.0 * (double)g[c];
            const float4 a = xv[r], b = xu[c];
            qs[0] += tg * ((double)a.x - (double)b.x);
            qs[1] += tg * ((double)a.y - (double)b.y);
            qs[2] += tg * ((double)a.z - (double)b.z);
            qs[3] += tg * ((double)a.w - (double)b.w);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qs[i] += __shfl_xor_sync(FG_FULL_MASK, qs[i], o);
        if (lane == 0 && p0 + r < n) two_sum_add(hi + v[r], lo + v[r], qs);
    }
}

// d == 4 (16-byte aligned float32 coordinates), k <= 65: a persistent warp
// walks its rows (i, i + W, ... in `order`) as a software pipeline -- the
// idx / upstream loads of row i+2 and the coordinate gathers of row i+1 are in
// flight while row i's terms are formed and its returning hi atomics issue,
// and the TwoSum corrections (lo REDs) of row i-1 go out once their atomics
// have returned.  The query side of a row (a warp sum, exactly one writer) is
// stored, not accumulated: qside[v].  Same arithmetic as k_knn_bwd_pipe.
#ifndef FG_BWD_CHUNK
#define FG_BWD_CHUNK 64
#endif
constexpr int kBwdChunk = FG_BWD_CHUNK;  // rows per CTA chunk (k_knn_bwd_stream)

struct BwdRow {
    int64_t v;
    int32_t u[2];
    float g[2];
};

__device__ __forceinline__ void bwd_load_row(BwdRow& r, int64_t i, int64_t n, const int32_t* __restrict__ order,
                                             const int32_t* __restrict__ idx, const float* __restrict__ gd2,
                                             int k) {
    const int lane = lane_id();
    r.v = i < n ? (order ? (int64_t)order[i] : i) : -1;
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const int s = 1 + lane + 32 * q;
        const bool ok = r.v >= 0 && s < k;
        r.u[q] = ok ? __ldcs(idx + r.v * k + s) : -1;  // streamed once: evict first
        r.g[q] = ok ? __ldcs(gd2 + r.v * k + s) : 0.0f;
    }
}

__global__ void __launch_bounds__(kRowWarps * 32) k_knn_bwd_stream(
    const float4* __restrict__ c4, int64_t n, const int32_t* __restrict__ idx, int k,
    const float* __restrict__ gd2, const int32_t* __restrict__ order, float4* __restrict__ hi,
    float4* __restrict__ lo, double4* __restrict__ qside) {
    const int lane = lane_id();
    // rows in chunks of kBwdChunk consecutive positions of the visiting order,
    // dealt round-robin to the CTAs: a CTA's warps work on spatial neighbours
    // (their neighbour gathers hit L1) and the rows in flight GPU-wide stay in
    // one window of the order (the atomics' targets stay L2-resident)
    constexpr int kPer = kBwdChunk / kRowWarps;  // rows per warp per chunk
    const int j = threadIdx.x >> 5;
    const int64_t G = gridDim.x;
    auto row_of = [&](int64_t t) -> int64_t {
        return ((int64_t)blockIdx.x + G * (t / kPer)) * kBwdChunk + j + kRowWarps * (t % kPer);
    };
    BwdRow r0, r1, r2;
    float4 xv0, xu0[2], xv1, xu1[2];
    auto gather = [&](const BwdRow& r, float4& xv, float4 (&xu)[2]) {
        xv = r.v >= 0 ? c4[r.v] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int q = 0; q < 2; ++q) xu[q] = r.u[q] >= 0 ? c4[r.u[q]] : xv;
    };
    bwd_load_row(r0, row_of(0), n, order, idx, gd2, k);
    bwd_load_row(r1, row_of(1), n, order, idx, gd2, k);
    gather(r0, xv0, xu0);
    // the previous row's pending corrections
    int32_t pu[2] = {-1, -1};
    float4 ph[2], pold[2];
    double px[2][4];
    for (int64_t t = 0; row_of(t) < n; ++t) {
        bwd_load_row(r2, row_of(t + 2), n, order, idx, gd2, k);
        gather(r1, xv1, xu1);
        // row i: exact float64 terms, returning hi atomics
        float4 h[2], old[2];
        double x[2][4];
        double qs[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const double tg = 2.0 * (double)r0.g[q];
            const float4 a = xv0, b = xu0[q];
            x[q][0] = tg * ((double)a.x - (double)b.x);
            x[q][1] = tg * ((double)a.y - (double)b.y);
            x[q][2] = tg * ((double)a.z - (double)b.z);
            x[q][3] = tg * ((double)a.w - (double)b.w);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                qs[e] += x[q][e];
                x[q][e] = -x[q][e];
            }
            h[q] = make_float4((float)x[q][0], (float)x[q][1], (float)x[q][2], (float)x[q][3]);
            if (r0.u[q] >= 0) old[q] = atomicAdd(hi + r0.u[q], h[q]);
        }
        // row i-1: corrections (their atomics have returned by now)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (pu[q] < 0) continue;
            const float* hp = &ph[q].x;
            const float* op = &pold[q].x;
            float4 l;
            float* lp = &l.x;
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                lp[e] = (float)(px[q][e] - (double)hp[e]);
                const float a2 = op[e], b2 = hp[e];
                const float sum = __fadd_rn(a2, b2);
                const float bb = __fsub_rn(sum, a2);
                const float err = __fadd_rn(__fsub_rn(a2, __fsub_rn(sum, bb)), __fsub_rn(b2, bb));
                lp[e] = isfinite(sum) ? __fadd_rn(lp[e], err) : 0.f;
            }
            atomicAdd(lo + pu[q], l);
        }
        // row i: the query side, stored by its one writer
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) qs[e] += __shfl_xor_sync(FG_FULL_MASK, qs[e], o);
        if (lane == 0 && r0.v >= 0) qside[r0.v] = make_double4(qs[0], qs[1], qs[2], qs[3]);
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            pu[q] = r0.u[q];
            ph[q] = h[q];
            pold[q] = old[q];
#pragma unroll
            for (int e = 0; e < 4; ++e) px[q][e] = x[q][e];
        }
        r0 = r1;
        xv0 = xv1;
        xu0[0] = xu1[0];
        xu0[1] = xu1[1];
        r1 = r2;
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {  // the last row's corrections
        if (pu[q] < 0) continue;
        const float* hp = &ph[q].x;
        const float* op = &pold[q].x;
        float4 l;
        float* lp = &l.x;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            lp[e] = (float)(px[q][e] - (double)hp[e]);
            const float a2 = op[e], b2 = hp[e];
            const float sum = __fadd_rn(a2, b2);
            const float bb = __fsub_rn(sum, a2);
            const float err = __fadd_rn(__fsub_rn(a2, __fsub_rn(sum, bb)), __fsub_rn(b2, bb));
            lp[e] = isfinite(sum) ? __fadd_rn(lp[e], err) : 0.f;
        }
        atomicAdd(lo + pu[q], l);
    }
}

__global__ void k_bwd_finish(const float4* __restrict__ hi, const float4* __restrict__ lo, int64_t n,
                             int n_c, int nv, void* __restrict__ out, int is_f64,
                             const double* __restrict__ qside) {
    const int64_t m = n * n_c;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = t / n_c;
        const int i = (int)(t - v * n_c);
        const float h = (&hi[v * nv + (i >> 2)].x)[i & 3];
        const float l = (&lo[v * nv + (i >> 2)].x)[i & 3];
        double x = (double)h + (double)l;
        if (qside) x += qside[v * 4 + i];
        if (is_f64)
            reinterpret_cast<double*>(out)[t] = x;
        else
            reinterpret_cast<float*>(out)[t] = (float)x;
    }
}

}  // namespace grad
}  // namespace fg

namespace fg {
namespace bt {

// destination bucket = 2^lb consecutive sorted positions (lb = 7 up to 2^21
// vertices, then growing so that at most kMaxBuckets buckets exist)
constexpr int kMinLB = 7;
constexpr int kMaxBuckets = 16384;
constexpr int64_t kMaxN = int64_t(1) << 23;  // src id (32 - lb bits) and dst offset share a word
constexpr int kWarps = 8;                    // count / scatter kernels: 256 threads
constexpr int kChunkBytes = 96 * 1024;       // counting-sort chunk of the reduce kernel

struct FastDiv {  // n / d for 32-bit n (Granlund-Montgomery, round-up multiplier)
    uint32_t d, m, sh;
    __host__ explicit FastDiv(uint32_t dd) : d(dd), m(0), sh(0) {
        uint32_t s = 0;
        while ((uint64_t(1) << s) < dd) ++s;
        if (dd > 1) {
            m = (uint32_t)(((uint64_t(1) << 32) * ((uint64_t(1) << s) - dd)) / dd + 1);
            sh = s - 1;
        }
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (d == 1) return n;
        const uint32_t t = __umulhi(n, m);
        return (t + ((n - t) >> 1)) >> sh;
    }
};

template <int NV>
__device__ __forceinline__ void load_row(const float* __restrict__ coords, int64_t w, int n_c, int vec4,
                                         float (&x)[4 * NV]) {
    if (NV == 1 && vec4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(coords) + w);
        x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
        return;
    }
#pragma unroll
    for (int i = 0; i < 4 * NV; ++i) x[i] = i < n_c ? __ldg(coords + w * n_c + i) : 0.f;
}

// biased exponent field of a double (0 for zero / subnormal, 0x7ff non-finite)
__device__ __forceinline__ int exp_field(double t) {
    return (int)((__double_as_longlong(t) >> 52) & 0x7ff);
}

__global__ void k_inv(const int32_t* __restrict__ order, int64_t n, int32_t* __restrict__ inv) {
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        inv[order[p]] = (int32_t)p;
}

// Sum of M = 2^m float64 values across the warp by transposition: log2(M)
// exchange steps halve the values each lane keeps, the remaining offsets
// reduce one value.  Lane L ends with the sum for index treduce_index(L), in a
// fixed order: deterministic.
template <int M>
__device__ __forceinline__ double treduce(double (&a)[M]) {
    const int lane = lane_id();
    int o = 16;
#pragma unroll
    for (int h = M / 2; h >= 1; h /= 2, o /= 2) {
        const bool hi = lane & o;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = hi ? a[i] : a[i + h];
            const double keep = hi ? a[i + h] : a[i];
            a[i] = keep + __shfl_xor_sync(FG_FULL_MASK, send, o);
        }
    }
    double r = a[0];
    for (; o >= 1; o /= 2) r += __shfl_xor_sync(FG_FULL_MASK, r, o);
    return r;
}
template <int M>
__device__ __forceinline__ int treduce_index(int lane) {
    int j = 0, o = 16;
#pragma unroll
    for (int h = M / 2; h >= 1; h /= 2, o /= 2) j += (lane & o) ? h : 0;
    return j;
}
template <int M>
__device__ __forceinline__ bool treduce_writer(int lane) {  // one lane per sum
    return (lane & (32 / M - 1)) == 0;
}

// K7a: entries per destination bucket.  Blocks of kRowsPerBlock consecutive
// sorted rows (their neighbours fall into few buckets: few (block, bucket)
// pairs, long runs), the block's (k-1)-slot entries walked flat over the CTA
// with the loads of 8 entries per thread in flight; shared-memory histogram,
// touched list, one global add per (block, touched bucket).
constexpr int kRowsPerBlock = 1024;
__global__ void __launch_bounds__(kWarps * 32) k_bt_count(const int32_t* __restrict__ idx, int64_t n, int k,
                                                       FastDiv divkm1, const int32_t* __restrict__ order,
                                                       const int32_t* __restrict__ inv, int lb, int n_buckets,
                                                       uint32_t* __restrict__ counts) {
    extern __shared__ uint32_t s_cnt[];
    uint32_t* s_hist = s_cnt;
    uint32_t* s_touched = s_cnt + n_buckets;
    int32_t* s_rows = reinterpret_cast<int32_t*>(s_touched + n_buckets);
    __shared__ uint32_t s_nt;
    for (int i = threadIdx.x; i < n_buckets; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x == 0) s_nt = 0;
    __syncthreads();
    const int64_t n_blocks = ceil_div(n, (int64_t)kRowsPerBlock);
    for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
        const int64_t p0 = blk * kRowsPerBlock;
        const int nr = (int)(n - p0 >= kRowsPerBlock ? kRowsPerBlock : n - p0);
        for (int r = threadIdx.x; r < nr; r += blockDim.x) s_rows[r] = order ? order[p0 + r] : (int32_t)(p0 + r);
        __syncthreads();
        const uint32_t m_tot = (uint32_t)nr * (uint32_t)(k - 1);
        for (uint32_t f0 = threadIdx.x; f0 < m_tot; f0 += 8 * kWarps * 32) {
            int32_t u[8];
            uint32_t pu[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t f = f0 + (uint32_t)j * (kWarps * 32);
                u[j] = -1;
                if (f < m_tot) {
                    const uint32_t r = divkm1.div(f);
                    u[j] = idx[(int64_t)s_rows[r] * k + 1 + (f - r * divkm1.d)];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) pu[j] = u[j] >= 0 ? (uint32_t)(inv ? inv[u[j]] : u[j]) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (u[j] >= 0) {
                    const uint32_t b = pu[j] >> lb;
                    if (atomicAdd(&s_hist[b], 1u) == 0) s_touched[atomicAdd(&s_nt, 1u)] = b;
                }
            }
        }
        __syncthreads();
        const uint32_t nt = s_nt;
        for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
            const uint32_t bb = s_touched[t];
            atomicAdd(&counts[bb], s_hist[bb]);
            s_hist[bb] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_nt = 0;
        __syncthreads();
    }
}

// K7c: the bucketed entries and the query side.  Same blocks as K7a.  Sweep 1
// counts the block's entries per bucket and claims a global range per touched
// bucket; sweep 2 (a half-warp per row, SPL slots per lane, every load in
// flight) forms the exact float64 terms -- the query side of the row is summed
// in a fixed order and written to qside[p] -- and writes one 8-byte entry per
// slot at its bucket range (rank from a shared-memory cursor).  The bucket's
// exponent bound is the block's largest term exponent.  Entry word: low 32
// bits = src id << lb | dst offset, high 32 bits = the upstream g (float bits).
template <int NV, int SPL>
__global__ void __launch_bounds__(kWarps * 32) k_bt_scatter(
    const float* __restrict__ coords, int n_c, int vec4, const int32_t* __restrict__ idx, int64_t n, int k,
    FastDiv divkm1, const float* __restrict__ gd2, const int32_t* __restrict__ order,
    const int32_t* __restrict__ inv, int lb, int n_buckets, uint32_t* __restrict__ cursor,
    int* __restrict__ emax_g, unsigned long long* __restrict__ entries, double* __restrict__ qside) {
    constexpr int NC = 4 * NV;
    constexpr int M = 2 * NC <= 8 ? 8 : (2 * NC <= 16 ? 16 : 32);
    extern __shared__ uint32_t s_sc[];
    uint32_t* s_hist = s_sc;
    uint32_t* s_touched = s_sc + n_buckets;
    int32_t* s_rows = reinterpret_cast<int32_t*>(s_touched + n_buckets);
    __shared__ uint32_t s_nt;
    __shared__ int s_emax;
    const int lane = lane_id(), w = threadIdx.x >> 5, hl = lane & 15, half = lane >> 4;
    for (int i = threadIdx.x; i < n_buckets; i += blockDim.x) s_hist[i] = 0;
    if (threadIdx.x == 0) {
        s_nt = 0;
        s_emax = 0;
    }
    __syncthreads();
    const int64_t n_blocks = ceil_div(n, (int64_t)kRowsPerBlock);
    const uint32_t mask = (1u << lb) - 1;
    for (int64_t blk = blockIdx.x; blk < n_blocks; blk += gridDim.x) {
        const int64_t p0 = blk * kRowsPerBlock;
        const int nr = (int)(n - p0 >= kRowsPerBlock ? kRowsPerBlock : n - p0);
        for (int r = threadIdx.x; r < nr; r += blockDim.x) s_rows[r] = order ? order[p0 + r] : (int32_t)(p0 + r);
        __syncthreads();
        // sweep 1: counts
        const uint32_t m_tot = (uint32_t)nr * (uint32_t)(k - 1);
        for (uint32_t f0 = threadIdx.x; f0 < m_tot; f0 += 8 * kWarps * 32) {
            int32_t u[8];
            uint32_t pu[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t f = f0 + (uint32_t)j * (kWarps * 32);
                u[j] = -1;
                if (f < m_tot) {
                    const uint32_t r = divkm1.div(f);
                    u[j] = idx[(int64_t)s_rows[r] * k + 1 + (f - r * divkm1.d)];
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) pu[j] = u[j] >= 0 ? (uint32_t)(inv ? inv[u[j]] : u[j]) : 0u;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (u[j] >= 0) {
                    const uint32_t b = pu[j] >> lb;
                    if (atomicAdd(&s_hist[b], 1u) == 0) s_touched[atomicAdd(&s_nt, 1u)] = b;
                }
            }
        }
        __syncthreads();
        const uint32_t nt = s_nt;
        for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
            const uint32_t b = s_touched[t];
            s_hist[b] = atomicAdd(&cursor[b], s_hist[b]);  // count -> global base (cursor)
        }
        __syncthreads();
        // sweep 2: half-warp per row
        int mexp = 0;
        for (int r0 = 2 * w; r0 < nr; r0 += 2 * kWarps) {
            const int r = r0 + half;
            const bool rv = r < nr;
            const int64_t v = rv ? s_rows[r] : 0;
            float xv[NC];
            load_row<NV>(coords, v, n_c, vec4, xv);
            double qa[NC];  // this half's row
#pragma unroll
            for (int i = 0; i < NC; ++i) qa[i] = 0.0;
            for (int sb = 1; sb < k; sb += 16 * SPL) {
                int32_t u[SPL];
                float g[SPL];
#pragma unroll
                for (int q = 0; q < SPL; ++q) {
                    const int s = sb + hl + 16 * q;
                    const bool ok = rv && s < k;
                    u[q] = ok ? idx[v * k + s] : -1;
                    g[q] = ok ? gd2[v * k + s] : 0.f;
                }
                float xu[SPL][NC];
                uint32_t pu[SPL];
#pragma unroll
                for (int q = 0; q < SPL; ++q) {
                    load_row<NV>(coords, u[q] >= 0 ? u[q] : v, n_c, vec4, xu[q]);
                    pu[q] = u[q] >= 0 ? (uint32_t)(inv ? inv[u[q]] : u[q]) : 0u;
                }
#pragma unroll
                for (int q = 0; q < SPL; ++q) {
                    if (u[q] < 0) continue;
                    const double tg = 2.0 * (double)g[q];
#pragma unroll
                    for (int i = 0; i < NC; ++i) {
                        if (i < n_c) {
                            const double t = tg * ((double)xv[i] - (double)xu[q][i]);  // exact
                            qa[i] += t;
                            const int be = exp_field(t);
                            if (be != 0x7ff) mexp = max(mexp, be);
                        }
                    }
                    const uint32_t b = pu[q] >> lb;
                    entries[atomicAdd(&s_hist[b], 1u)] =
                        ((unsigned long long)__float_as_uint(g[q]) << 32) | (((uint32_t)v << lb) | (pu[q] & mask));
                }
            }
            // the two rows' query sides: lanes of the other half contribute zeros
            double qs[M];
#pragma unroll
            for (int i = 0; i < M; ++i) qs[i] = 0.0;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                qs[i] = half ? 0.0 : qa[i];
                qs[NC + i] = half ? qa[i] : 0.0;
            }
            const double sum = treduce<M>(qs);
            if (treduce_writer<M>(lane)) {
                const int j = treduce_index<M>(lane);
                const int rr = r0 + j / NC, i = j % NC;
                if (j < 2 * NC && rr < nr && i < n_c) qside[(p0 + rr) * n_c + i] = sum;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mexp = max(mexp, __shfl_xor_sync(FG_FULL_MASK, mexp, o));
        if (lane == 0) atomicMax(&s_emax, mexp);
        __syncthreads();
        const int cemax = s_emax;
        for (uint32_t t = threadIdx.x; t < nt; t += blockDim.x) {
            atomicMax(&emax_g[s_touched[t]], cemax);
            s_hist[s_touched[t]] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_nt = 0;
            s_emax = 0;
        }
        __syncthreads();
    }
}

// K7d: CTA per destination bucket, thread per destination (blockDim = 2^lb).
// Per chunk of the bucket's entries: histogram by destination, scan, rank ->
// payloads in destination order in shared memory, then every thread sums its
// destination's terms as int64 multiples of the bucket quantum 2^q (exact
// integer addition: the result does not depend on the order entries arrived
// in), and finally adds the query side.
template <int NV>
__global__ void __launch_bounds__(512, 2) k_bt_reduce(
    const float* __restrict__ coords, int64_t n, int n_c, int vec4, const int32_t* __restrict__ order, int lb,
    const uint32_t* __restrict__ offsets, const int* __restrict__ emax_g,
    const unsigned long long* __restrict__ entries, const double* __restrict__ qside,
    void* __restrict__ out, int is_f64, int chunk) {
    constexpr int NC = 4 * NV;
    constexpr int BW = NV == 1 ? 4 : 2;  // gathers in flight per thread
    extern __shared__ __align__(16) unsigned long long s_sorted[];
    __shared__ uint32_t s_hist[512];
    __shared__ uint32_t s_cur[512];
    __shared__ uint32_t s_wsum[16];
    const int nt = blockDim.x;  // = 2^lb
    const int t = threadIdx.x, lane = lane_id(), w = t >> 5;
    const int64_t b = blockIdx.x;
    const int64_t p = (b << lb) + t;
    const bool live = p < n;
    const int64_t u = live ? (order ? (int64_t)order[p] : p) : 0;
    float xu[NC];
    load_row<NV>(coords, u, n_c, vec4, xu);
    const uint32_t off = offsets[b];
    const uint32_t cnt = offsets[b + 1] - off;
    const unsigned long long* src = entries + off;
    const uint32_t mask = (uint32_t)nt - 1;
    // quantum 2^q: |term| < 2^emax, at most cnt terms -> |sum| < 2^62 in units of 2^q
    const int emax = max(emax_g[b], 1) - 1022;
    const int l2e = 32 - __clz(cnt + 1);
    const int q = max(emax + l2e - 62, -1022);
    const double pw = __longlong_as_double((long long)(1023 - q) << 52);    // 2^-q
    const double pwinv = __longlong_as_double((long long)(1023 + q) << 52);  // 2^q
    long long acc[NC];
    double nf[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        acc[i] = 0;
        nf[i] = 0.0;
    }
    const int nwarps = nt >> 5;
    for (uint32_t c0 = 0; c0 < cnt; c0 += chunk) {
        const uint32_t m = min((uint32_t)chunk, cnt - c0);
        s_hist[t] = 0;
        __syncthreads();
        for (uint32_t e0 = t; e0 < m; e0 += 8 * nt) {
            uint32_t dl[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) dl[j] = e0 + j * nt < m ? (uint32_t)src[c0 + e0 + j * nt] & mask : 0xffffffffu;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (dl[j] != 0xffffffffu) atomicAdd(&s_hist[dl[j]], 1u);
        }
        __syncthreads();
        const uint32_t h = s_hist[t];
        const uint32_t incl = warp_inclusive_scan(h);
        if (lane == 31) s_wsum[w] = incl;
        __syncthreads();
        if (w == 0) {
            uint32_t x = lane < nwarps ? s_wsum[lane] : 0;
            x = warp_inclusive_scan(x);
            if (lane < nwarps) s_wsum[lane] = x;
        }
        __syncthreads();
        const uint32_t st = incl - h + (w > 0 ? s_wsum[w - 1] : 0);
        s_cur[t] = st;
        __syncthreads();
        for (uint32_t e0 = t; e0 < m; e0 += 8 * nt) {
            unsigned long long pay[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) pay[j] = e0 + j * nt < m ? src[c0 + e0 + j * nt] : ~0ull;
#pragma unroll
            for (int j = 0; j < 8; ++j)
                if (pay[j] != ~0ull) s_sorted[atomicAdd(&s_cur[(uint32_t)pay[j] & mask], 1u)] = pay[j];
        }
        __syncthreads();
        for (uint32_t i0 = st; i0 < st + h; i0 += BW) {
            unsigned long long pays[BW];
            float xv[BW][NC];
#pragma unroll
            for (int j = 0; j < BW; ++j) {
                pays[j] = i0 + j < st + h ? s_sorted[i0 + j] : 0ull;
                load_row<NV>(coords, i0 + j < st + h ? (int64_t)((uint32_t)pays[j] >> lb) : u, n_c, vec4, xv[j]);
            }
#pragma unroll
            for (int j = 0; j < BW; ++j) {
                if (i0 + j < st + h) {
                    const double tgq = 2.0 * (double)__uint_as_float((uint32_t)(pays[j] >> 32)) * pw;
#pragma unroll
                    for (int i = 0; i < NC; ++i) {
                        if (i < n_c) {
                            // -2g(x_v - x_u) in units of 2^q: exact (power-of-two scaling of an exact product)
                            const double term = tgq * ((double)xu[i] - (double)xv[j][i]);
                            if (exp_field(term) != 0x7ff)
                                acc[i] += __double2ll_rn(term);
                            else
                                nf[i] += term;
                        }
                    }
                }
            }
        }
        __syncthreads();
    }
    if (!live) return;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        if (i < n_c) {
            const double r = qside[p * n_c + i] + ((double)acc[i] * pwinv + nf[i] * pwinv);
            if (is_f64)
                reinterpret_cast<double*>(out)[u * n_c + i] = r;
            else
                reinterpret_cast<float*>(out)[u * n_c + i] = (float)r;
        }
    }
}

struct Plan {
    bool ok = false;
    int n_buckets = 0, nv = 1, lb = kMinLB, chunk = 0;
    size_t off_inv = 0, off_counts = 0, off_emax = 0, off_offsets = 0, off_cursor = 0, off_status = 0,
           off_ticket = 0, off_entries = 0, off_qside = 0, bytes = 0, blk_smem = 0, reduce_smem = 0,
           zero_lo = 0, zero_hi = 0;
    int64_t n_tiles = 0;
};

inline Plan plan(int64_t n, int n_c, int k) {
    Plan P;
    if (n < 1 || n > kMaxN || k < 1) return P;
    const int64_t slots = n * (int64_t)(k - 1);
    if (n * (int64_t)k >= (int64_t(1) << 32)) return P;
    P.nv = (n_c + 3) / 4;
    P.lb = 9;
    P.n_buckets = (int)ceil_div(n, int64_t(1) << P.lb);
    if (P.n_buckets > kMaxBuckets) return P;
    P.blk_smem = (size_t)P.n_buckets * 8 + (size_t)kRowsPerBlock * 4;
    P.chunk = (int)(kChunkBytes / 8);
    P.reduce_smem = (size_t)P.chunk * 8;
    P.n_tiles = ceil_div(P.n_buckets, kScanTile);
    size_t o = 0;
    auto take = [&](size_t bytes) {
        const size_t at = o;
        o = align_up(o + bytes, 256);
        return at;
    };
    P.off_inv = take((size_t)n * 4);
    P.zero_lo = o;
    P.off_counts = take((size_t)P.n_buckets * 4);
    P.off_emax = take((size_t)P.n_buckets * 4);
    P.off_status = take((size_t)P.n_tiles * 8);
    P.off_ticket = take(4);
    P.zero_hi = o;
    P.off_offsets = take((size_t)(P.n_buckets + 1) * 4);
    P.off_cursor = take((size_t)P.n_buckets * 4);
    P.off_entries = take((size_t)std::max<int64_t>(slots, 1) * 8);
    P.off_qside = take((size_t)n * n_c * 8);
    P.bytes = o;
    P.ok = true;
    return P;
}

template <int NV>
int launch(const Plan& P, const float* coords, int64_t n, int n_c, const int32_t* idx, int k,
           const float* gd2, const int32_t* order, void* out, int is_f64, char* ws, cudaStream_t st) {
    int dev = 0, sms = 148;
    FG_CUDA(cudaGetDevice(&dev));
    FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int vec4 = (n_c == 4 && (reinterpret_cast<uintptr_t>(coords) & 15) == 0) ? 1 : 0;
    int32_t* inv = nullptr;
    if (order) {
        inv = reinterpret_cast<int32_t*>(ws + P.off_inv);
        k_inv<<<(unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)sms * 8), 256, 0, st>>>(order, n, inv);
        FG_TRY(launched(st));
    }
    uint32_t* counts = reinterpret_cast<uint32_t*>(ws + P.off_counts);
    int* emax = reinterpret_cast<int*>(ws + P.off_emax);
    uint32_t* offsets = reinterpret_cast<uint32_t*>(ws + P.off_offsets);
    uint32_t* cursor = reinterpret_cast<uint32_t*>(ws + P.off_cursor);
    unsigned long long* entries = reinterpret_cast<unsigned long long*>(ws + P.off_entries);
    double* qside = reinterpret_cast<double*>(ws + P.off_qside);
    FG_CUDA(cudaMemsetAsync(ws + P.zero_lo, 0, P.zero_hi - P.zero_lo, st));
    const int64_t n_blocks = ceil_div(n, (int64_t)kRowsPerBlock);
    const FastDiv divkm1((uint32_t)std::max(k - 1, 1));
    if (k > 1) {
        FG_CUDA(cudaFuncSetAttribute(k_bt_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.blk_smem));
        int occ = 1;
        FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bt_count, kWarps * 32, P.blk_smem));
        k_bt_count<<<(unsigned)std::min<int64_t>(n_blocks, (int64_t)sms * std::max(occ, 1)), kWarps * 32,
                     P.blk_smem, st>>>(idx, n, k, divkm1, order, inv, P.lb, P.n_buckets, counts);
        FG_TRY(launched(st));
    }
    k_scan<<<(unsigned)P.n_tiles, kScanThreads, 0, st>>>(
        reinterpret_cast<const int32_t*>(counts), P.n_buckets, reinterpret_cast<int32_t*>(offsets),
        reinterpret_cast<int32_t*>(cursor), reinterpret_cast<unsigned long long*>(ws + P.off_status),
        reinterpret_cast<unsigned*>(ws + P.off_ticket));
    FG_TRY(launched(st));
    auto scatter = [&](auto kern) -> int {
        FG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.blk_smem));
        int occ = 1;
        FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kWarps * 32, P.blk_smem));
        kern<<<(unsigned)std::min<int64_t>(n_blocks, (int64_t)sms * std::max(occ, 1)), kWarps * 32, P.blk_smem,
               st>>>(coords, n_c, vec4, idx, n, k, divkm1, gd2, order, inv, P.lb, P.n_buckets, cursor, emax,
                     entries, qside);
        return launched(st);
    };
    if (k <= 17)
        FG_TRY(scatter(k_bt_scatter<NV, 1>));
    else if (k <= 33 || NV > 1)
        FG_TRY(scatter(k_bt_scatter<NV, 2>));
    else
        FG_TRY(scatter(k_bt_scatter<NV, 3>));
    FG_CUDA(cudaFuncSetAttribute(k_bt_reduce<NV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)P.reduce_smem));
    k_bt_reduce<NV><<<(unsigned)P.n_buckets, 1 << P.lb, P.reduce_smem, st>>>(
        coords, n, n_c, vec4, order, P.lb, offsets, emax, entries, qside, out, is_f64, P.chunk);
    return launched(st);
}

}  // namespace bt
}  // namespace fg

using namespace fg;
using namespace fg::grad;

namespace {
size_t fallback_bytes(int64_t n, int n_coords) {
    const int nv = (n_coords + 3) / 4;
    // hi, lo (float4 per 4 coordinates) + the streamed kernel's query sides (d == 4)
    return 2 * align_up(sizeof(float4) * (size_t)n * nv, 256) +
           (n_coords == 4 ? align_up(sizeof(double) * 4 * (size_t)n, 256) : 0);
}
}  // namespace

extern "C" int fg_knn_bwd_workspace_size(int64_t n, int32_t n_coords, int32_t k, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_coords < 1) return FG_ERR_BAD_SHAPE;
    if (k < 1) return FG_ERR_BAD_K;
    const bt::Plan P = bt::plan(n, n_coords, k);
    *bytes = std::max(P.ok ? P.bytes : 0, fallback_bytes(n, n_coords));  // either path
    if (*bytes == 0) *bytes = 256;
    return 0;
}

extern "C" int fg_knn_bwd(const void* coords_v, int64_t n, int32_t n_coords, const int32_t* idx,
                          int32_t k, const void* grad_v, const int32_t* order, void* grad_coords,
                          int32_t grad_flags, void* workspace, size_t workspace_bytes,
                          void* stream) {
    const bool x64 = grad_flags & FG_BWD_X64, g64 = grad_flags & FG_BWD_G64;
    const float* coords = static_cast<const float*>(coords_v);
    const float* grad_d2 = static_cast<const float*>(grad_v);
    const int grad_is_f64 = (grad_flags & FG_BWD_F64) ? 1 : 0;
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_coords < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords > 16) return FG_ERR_TOO_MANY_DIMS;
    if (n == 0) return 0;
    if (!coords || !idx || !grad_d2 || !grad_coords || !workspace) return FG_ERR_NULL;
    cudaStream_t st = (cudaStream_t)stream;
    const int nv = (n_coords + 3) / 4;
    const bt::Plan P = bt::plan(n, n_coords, k);
    if (grad_flags & FG_BWD_DETERMINISTIC) {
        if (!P.ok || x64 || g64) return FG_ERR_UNSUPPORTED;
        if (workspace_bytes < P.bytes) return FG_ERR_WORKSPACE;
        char* ws = static_cast<char*>(workspace);
        switch (nv) {
            case 1: return bt::launch<1>(P, coords, n, n_coords, idx, k, grad_d2, order, grad_coords, grad_is_f64, ws, st);
            case 2: return bt::launch<2>(P, coords, n, n_coords, idx, k, grad_d2, order, grad_coords, grad_is_f64, ws, st);
            case 3: return bt::launch<3>(P, coords, n, n_coords, idx, k, grad_d2, order, grad_coords, grad_is_f64, ws, st);
            default: return bt::launch<4>(P, coords, n, n_coords, idx, k, grad_d2, order, grad_coords, grad_is_f64, ws, st);
        }
    }
    // compensated fp32x4 atomics
    const size_t half = align_up(sizeof(float4) * (size_t)n * nv, 256);
    if (workspace_bytes < fallback_bytes(n, n_coords)) return FG_ERR_WORKSPACE;
    float4* hi = (float4*)workspace;
    float4* lo = (float4*)((char*)workspace + half);
    double* qside = nullptr;
    FG_CUDA(cudaMemsetAsync(workspace, 0, 2 * half, st));
    const unsigned blocks = (unsigned)ceil_div(n, kRowWarps);
    const bool vec4 = n_coords == 4 && (reinterpret_cast<uintptr_t>(coords) & 15) == 0;
#ifndef FG_BWD_STREAM
#define FG_BWD_STREAM 1
#endif
    if (FG_BWD_STREAM && !x64 && !g64 && vec4 && k <= 65) {
        qside = (double*)((char*)workspace + 2 * half);
        int dev = 0, sms = 0, per_sm = 1;
        FG_CUDA(cudaGetDevice(&dev));
        FG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        FG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_knn_bwd_stream, kRowWarps * 32, 0));
        const int64_t grid = std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), blocks);
        k_knn_bwd_stream<<<(unsigned)grid, kRowWarps * 32, 0, st>>>(
            reinterpret_cast<const float4*>(coords), n, idx, k, grad_d2, order, hi, lo,
            reinterpret_cast<double4*>(qside));
    } else if (x64 || g64) {
        const double* c64 = static_cast<const double*>(coords_v);
        const double* g64p = static_cast<const double*>(grad_v);
#define FG_BWD_GEN(NVV)                                                                              \
    if (x64 && g64)                                                                                  \
        k_knn_bwd<NVV, double, double><<<blocks, kRowWarps * 32, 0, st>>>(c64, n, n_coords, idx, k, g64p, order, hi, lo); \
    else if (x64)                                                                                    \
        k_knn_bwd<NVV, double, float><<<blocks, kRowWarps * 32, 0, st>>>(c64, n, n_coords, idx, k, grad_d2, order, hi, lo); \
    else                                                                                             \
        k_knn_bwd<NVV, float, double><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, g64p, order, hi, lo);
        switch (nv) {
            case 1: FG_BWD_GEN(1) break;
            case 2: FG_BWD_GEN(2) break;
            case 3: FG_BWD_GEN(3) break;
            default: FG_BWD_GEN(4) break;
        }
#undef FG_BWD_GEN
    } else if (vec4 && k <= 33) {
        k_knn_bwd_pipe<1, 1><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo);
    } else if (vec4 && k <= 65) {
        k_knn_bwd_pipe<1, 2><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo);
    } else switch (nv) {
        case 1: k_knn_bwd<1, float, float><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        case 2: k_knn_bwd<2, float, float><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        case 3: k_knn_bwd<3, float, float><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        default: k_knn_bwd<4, float, float><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
    }
    FG_TRY(launched(st));
    const int64_t m = n * n_coords;
    k_bwd_finish<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 148 * 16), 256, 0, st>>>(
        hi, lo, n, n_coords, nv, grad_coords, grad_is_f64, qside);
    return launched(st);
}
