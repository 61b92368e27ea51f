// fg_gravnet.cu -- GravNet distance-weighted aggregation (replaces
// G/gravnet.py:64-150) for sm_100a.
//
// Semantics (G/gravnet.py): slot s of row v contributes when idx[v,s] >= 0 (and
// s > 0 unless include_self) with weight w = exp(-scale * d2[v,s]); reducers
// are applied in order, one F-wide block each: mean = sum / count over valid
// slots, max over valid slots (the backward routes it to the lowest arg-max
// slot, np.argmax), zeros for a row without valid slots.  Weights, products,
// sums and maxima are float64, outputs float32.
//
// Every pass is a gather of feature-sized rows (256 B for F = 64) indexed by
// the neighbour matrix, so the kernels are built for memory-level
// parallelism: a warp owns a row, each lane VW consecutive features (one
// float2/float4 load per gathered row), and the slots are taken U = 8 at a
// time with all U gathers issued before any arithmetic.  Rows are visited in
// `order` when given: spatially sorted rows share most of their neighbours,
// so consecutive warps hit the same feature rows in L1/L2.
//
// Backward:
//   rows    warp per row v: per-feature arg-max slot (registers), grad_d2[v,s] =
//           -scale w_s sum_f f[u_s,f] coef[v,f,s] (the U per-slot dot products
//           of a batch are reduced together by a transposing butterfly: 9
//           shuffles instead of 5 U), the mean coefficients cm[v,f] =
//           sum_mean up/cnt_v, and the max-block gradient w cmax[v,f] sent to
//           the arg-max neighbour -- one float64 atomic per (v,f), N*F in all,
//           spread over N*F targets (not the k-fold scatter of the mean part);
//   reverse counting sort of the (v,s) pairs by neighbour u (int atomics +
//           the decoupled-look-back scan) -> for every u the list of (v,s)
//           that aggregated it;
//   columns warp per u gathers grad_feats[u,f] = gmax[u,f] + sum over its list
//           of w_vs cm[v,f], float64: one 4F-byte row and two FMAs per entry.
#include "fg_common.cuh"
#include "fg_scan.cuh"

#include <initializer_list>

namespace fg {
namespace gravnet {

constexpr int kRowWarps = 8;
constexpr int U = 8;  // gathers in flight per warp

struct GnArgs {
    const float* feats;
    int64_t n;
    int F;
    const int32_t* idx;
    const float* d2;
    int k;
    double scale;
    unsigned max_bits;  // bit b set: reducer block b is max (else mean)
    int n_red;
    int include_self;
    const int32_t* order;
};

__device__ __forceinline__ int64_t row_of(const GnArgs& g, int64_t p) {
    return g.order ? (int64_t)g.order[p] : p;
}

__device__ __forceinline__ bool is_max(const GnArgs& g, int b) { return (g.max_bits >> b) & 1u; }

__device__ __forceinline__ bool slot_valid(const GnArgs& g, int s, int32_t u) {
    return u >= 0 && (g.include_self || s > 0);
}

template <int VW>
__device__ __forceinline__ void ldf(const float* p, float (&x)[VW]) {
    if constexpr (VW == 4) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        x[0] = t.x; x[1] = t.y; x[2] = t.z; x[3] = t.w;
    } else if constexpr (VW == 2) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        x[0] = t.x; x[1] = t.y;
    } else {
        x[0] = __ldg(p);
    }
}

template <int VW>
__device__ __forceinline__ void stf(float* p, const float (&x)[VW]) {
    if constexpr (VW == 4)
        *reinterpret_cast<float4*>(p) = make_float4(x[0], x[1], x[2], x[3]);
    else if constexpr (VW == 2)
        *reinterpret_cast<float2*>(p) = make_float2(x[0], x[1]);
    else
        *p = x[0];
}

// Slot data of one 32-slot window: lane j holds slot base + j.
struct Window {
    int32_t u;
    double w;
    unsigned okm;
};

__device__ __forceinline__ Window load_window(const GnArgs& g, int64_t v, int base, bool weights) {
    const int lane = lane_id();
    const int s = base + lane;
    Window wd;
    wd.u = s < g.k ? __ldg(&g.idx[v * g.k + s]) : -1;
    const bool ok = s < g.k && slot_valid(g, s, wd.u);
    wd.w = ok && weights ? exp(-g.scale * (double)__ldg(&g.d2[v * g.k + s])) : 0.0;
    wd.okm = __ballot_sync(FG_FULL_MASK, ok);
    return wd;
}

// Gather UU slots' feature vectors (warp-uniform validity).
template <int VW, int UU = U>
__device__ __forceinline__ void gather(const GnArgs& g, const Window& wd, int j0, int fl, bool lane_on,
                                       float (&x)[UU][VW], double (&w)[UU], bool (&valid)[UU]) {
#pragma unroll
    for (int q = 0; q < UU; ++q) {
        const int jj = j0 + q;
        valid[q] = jj < 32 && ((wd.okm >> (jj & 31)) & 1u);
        const int32_t uq = __shfl_sync(FG_FULL_MASK, wd.u, jj & 31);
        w[q] = __shfl_sync(FG_FULL_MASK, wd.w, jj & 31);
#pragma unroll
        for (int e = 0; e < VW; ++e) x[q][e] = 0.0f;
        if (valid[q] && lane_on) ldf<VW>(g.feats + (int64_t)uq * g.F + fl, x[q]);
    }
}

// ---------------------------------------------------------------- forward
#ifndef FG_GN_FWD_U
#define FG_GN_FWD_U 4
#endif
template <int VW, int UF>
__device__ __forceinline__ void gn_fwd_row(const GnArgs& g, int f0, float* __restrict__ out, int64_t p) {
    const int lane = lane_id();
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const int fl = f0 + lane * VW;
    const bool lane_on = fl < F;
    double sum[VW], mx[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        sum[e] = 0.0;
        mx[e] = -INFINITY;
    }
    int cnt = 0;
    for (int base = 0; base < k; base += 32) {
        const Window wd = load_window(g, v, base, true);
        cnt += __popc(wd.okm);
        for (int j0 = 0; j0 < 32; j0 += UF) {
            if (((wd.okm >> j0) & (UF == 32 ? 0xffffffffu : ((1u << UF) - 1u))) == 0) continue;
            float x[UF][VW];
            double w[UF];
            bool valid[UF];
            gather<VW, UF>(g, wd, j0, fl, lane_on, x, w, valid);
#pragma unroll
            for (int q = 0; q < UF; ++q) {
                if (!valid[q]) continue;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const double term = w[q] * (double)x[q][e];
                    sum[e] += term;
                    mx[e] = term > mx[e] ? term : mx[e];
                }
            }
        }
    }
    if (!lane_on) return;
    for (int b = 0; b < g.n_red; ++b) {
        float o[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) o[e] = cnt > 0 ? (float)(is_max(g, b) ? mx[e] : sum[e] / (double)cnt) : 0.0f;
        stf<VW>(out + v * W + (int64_t)b * F + fl, o);
    }
}

template <int VW>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_fwd(const GnArgs g, int f0, float* __restrict__ out) {
    constexpr int UF = FG_GN_FWD_U;  // gathers in flight per warp
    const int lane = lane_id();
    const int64_t n_rows = g.n;
    for (int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5); p < n_rows;
         p += (int64_t)gridDim.x * kRowWarps)
        gn_fwd_row<VW, UF>(g, f0, out, p);
}

// Half-warp slot pairs (F % 4 == 0, F <= 64): lanes 0-15 take slot j, lanes
// 16-31 slot j+1, each lane 4 features (one 16-byte gather), so the per-slot
// bookkeeping (neighbour id / weight shuffles, validity, address) is paid by
// half the lanes per feature; the two halves are combined at the end.
#ifndef FG_GN_PAIRS_U
#define FG_GN_PAIRS_U 2
#endif

template <int UP>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_fwd_pairs(const GnArgs g, float* __restrict__ out) {
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const int half = lane >> 4;
    const int fl = (lane & 15) * 4;
    const bool lane_on = fl < F;
    double sum[4], mx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sum[e] = 0.0;
        mx[e] = -INFINITY;
    }
    int cnt = 0;
    for (int base = 0; base < k; base += 32) {
        const Window wd = load_window(g, v, base, true);
        cnt += __popc(wd.okm);
        for (int j0 = 0; j0 < 32; j0 += 2 * UP) {
            if (((wd.okm >> j0) & ((1u << (2 * UP)) - 1u)) == 0) continue;
            float4 x[UP];
            double w[UP];
            bool valid[UP];
#pragma unroll
            for (int q = 0; q < UP; ++q) {
                const int jj = j0 + 2 * q + half;
                valid[q] = (wd.okm >> jj) & 1u;
                const int32_t uq = __shfl_sync(FG_FULL_MASK, wd.u, jj);
                w[q] = __shfl_sync(FG_FULL_MASK, wd.w, jj);
                x[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (valid[q] && lane_on)
                    x[q] = __ldg(reinterpret_cast<const float4*>(g.feats + (int64_t)uq * F + fl));
            }
#pragma unroll
            for (int q = 0; q < UP; ++q) {
                if (!valid[q]) continue;
                const float xe[4] = {x[q].x, x[q].y, x[q].z, x[q].w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const double term = w[q] * (double)xe[e];
                    sum[e] += term;
                    mx[e] = term > mx[e] ? term : mx[e];
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        sum[e] += __shfl_xor_sync(FG_FULL_MASK, sum[e], 16);
        const double om = __shfl_xor_sync(FG_FULL_MASK, mx[e], 16);
        mx[e] = om > mx[e] ? om : mx[e];  // the value; which slot holds it does not matter here
    }
    if (half || !lane_on) return;
    for (int b = 0; b < g.n_red; ++b) {
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = cnt > 0 ? (float)(is_max(g, b) ? mx[e] : sum[e] / (double)cnt) : 0.0f;
        *reinterpret_cast<float4*>(out + v * W + (int64_t)b * F + fl) = make_float4(o[0], o[1], o[2], o[3]);
    }
}

// ---------------------------------------------------------------- backward
struct GnBwd {
    const float* up;      // (n, F * n_red)
    float* cm;            // (n, F) mean-block coefficient sum_b up_b / cnt (0: no valid slot)
    double* gmax;         // (n, F) max-block gradient, scattered to the arg-max neighbour; null: no max
    float* grad_d2;       // (n, k)
    double* gd_acc;       // (n, k) float64 partials when F spans several chunks, else null
    int32_t* rev_cnt;     // (n) reverse-neighbour counts (scan input)
    int32_t* rev_off;     // (n + 1)
    int32_t* rev_cur;     // (n) fill cursor
    int32_t* rev;         // (n * k) entries v * k + s
    float* grad_feats;    // (n, F)
    int has_mean;
};

// Sum a[q] over the warp for q = 0..7 at once; lane L ends with the total of
// q = 4 b4 + 2 b3 + b2 (bits of L).  5 shuffle rounds, 4 + 2 + 1 + 1 + 1 values.
__device__ __forceinline__ double transpose_reduce8(double (&a)[8]) {
    const int lane = lane_id();
    {
        const bool hi = lane & 16;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const double send = hi ? a[i] : a[i + 4];
            const double keep = hi ? a[i + 4] : a[i];
            a[i] = keep + __shfl_xor_sync(FG_FULL_MASK, send, 16);
        }
    }
    {
        const bool hi = lane & 8;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double send = hi ? a[i] : a[i + 2];
            const double keep = hi ? a[i + 2] : a[i];
            a[i] = keep + __shfl_xor_sync(FG_FULL_MASK, send, 8);
        }
    }
    {
        const bool hi = lane & 4;
        const double send = hi ? a[0] : a[1];
        const double keep = hi ? a[1] : a[0];
        a[0] = keep + __shfl_xor_sync(FG_FULL_MASK, send, 4);
    }
    double r = a[0];
    r += __shfl_xor_sync(FG_FULL_MASK, r, 2);
    r += __shfl_xor_sync(FG_FULL_MASK, r, 1);
    return r;
}

__device__ __forceinline__ int reduce8_src(int q) { return ((q >> 2) & 1) << 4 | ((q >> 1) & 1) << 3 | (q & 1) << 2; }

// Sum a[q] over the warp for q = 0..3 at once; lane L ends with the total of
// q = 2 b4 + b3 (bits of L).
__device__ __forceinline__ double transpose_reduce4(double (&a)[4]) {
    const int lane = lane_id();
    {
        const bool hi = lane & 16;
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const double send = hi ? a[i] : a[i + 2];
            const double keep = hi ? a[i + 2] : a[i];
            a[i] = keep + __shfl_xor_sync(FG_FULL_MASK, send, 16);
        }
    }
    {
        const bool hi = lane & 8;
        const double send = hi ? a[0] : a[1];
        const double keep = hi ? a[1] : a[0];
        a[0] = keep + __shfl_xor_sync(FG_FULL_MASK, send, 8);
    }
    double r = a[0];
    r += __shfl_xor_sync(FG_FULL_MASK, r, 4);
    r += __shfl_xor_sync(FG_FULL_MASK, r, 2);
    r += __shfl_xor_sync(FG_FULL_MASK, r, 1);
    return r;
}

__device__ __forceinline__ int reduce4_src(int q) { return ((q >> 1) & 1) << 4 | (q & 1) << 3; }

// Row pass: arg-max slots (registers), grad_d2, the mean coefficients cm and
// the max-block gradients (float64 atomics, one per (v, f) to its arg-max
// neighbour); counts reverse neighbours.
template <int VW>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_rows(const GnArgs g, const GnBwd bw, int f0,
                                                          int last_chunk) {
    static_assert(U == 8, "transpose_reduce8");
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const int fl = f0 + lane * VW;
    const bool lane_on = fl < F;
    const bool has_max = g.max_bits != 0;
    // pass 1: count (+ reverse counts) and arg-max (lowest slot on ties, np.argmax)
    int cnt = 0;
    double best[VW];
    int bslot[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        best[e] = -INFINITY;
        bslot[e] = -1;
    }
    for (int base = 0; base < k; base += 32) {
        const Window wd = load_window(g, v, base, has_max);
        cnt += __popc(wd.okm);
        if (f0 == 0 && ((wd.okm >> lane) & 1u)) atomicAdd(&bw.rev_cnt[wd.u], 1);
        if (!has_max) continue;
        for (int j0 = 0; j0 < 32; j0 += U) {
            if (((wd.okm >> j0) & ((1u << U) - 1u)) == 0) continue;
            float x[U][VW];
            double w[U];
            bool valid[U];
            gather<VW>(g, wd, j0, fl, lane_on, x, w, valid);
#pragma unroll
            for (int q = 0; q < U; ++q) {
                if (!valid[q]) continue;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const double term = w[q] * (double)x[q][e];
                    if (term > best[e]) {
                        best[e] = term;
                        bslot[e] = base + j0 + q;
                    }
                }
            }
        }
    }
    // per-feature coefficients: mean blocks up/cnt, max blocks up at the arg-max
    double cmean[VW], cmax[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        cmean[e] = 0.0;
        cmax[e] = 0.0;
    }
    if (lane_on && cnt > 0) {
        for (int b = 0; b < g.n_red; ++b) {
            float ub[VW];
            ldf<VW>(bw.up + v * W + (int64_t)b * F + fl, ub);
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                if (is_max(g, b))
                    cmax[e] += (double)ub[e];
                else
                    cmean[e] += (double)ub[e] / (double)cnt;
            }
        }
    }
    if (lane_on && bw.has_mean) {
        float o[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) o[e] = (float)cmean[e];
        stf<VW>(bw.cm + v * F + fl, o);
    }
    // pass 2: grad_d2[v,s] = -scale w_s sum_f f[u_s,f] (cmean_f + [amax_f == s] cmax_f);
    // the max blocks' feature gradient w_s cmax_f goes to u_s at s = amax_f
    for (int base = 0; base < k; base += 32) {
        const Window wd = load_window(g, v, base, true);
        const unsigned okm = cnt > 0 ? wd.okm : 0u;
        double mine = 0.0;  // this lane's slot total
        for (int j0 = 0; j0 < 32; j0 += U) {
            if (((okm >> j0) & ((1u << U) - 1u)) == 0) continue;
            float x[U][VW];
            double w[U];
            bool valid[U];
            gather<VW>(g, wd, j0, fl, lane_on, x, w, valid);
            double part[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                part[q] = 0.0;
                const int32_t uq = __shfl_sync(FG_FULL_MASK, wd.u, (j0 + q) & 31);
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    const bool at = bslot[e] == base + j0 + q;
                    const double c = cmean[e] + (at ? cmax[e] : 0.0);
                    part[q] += (double)x[q][e] * c;
                    if (at && lane_on && bw.gmax) atomicAdd(&bw.gmax[(int64_t)uq * F + fl + e], w[q] * cmax[e]);
                }
            }
            const double r = transpose_reduce8(part);
            const double got = __shfl_sync(FG_FULL_MASK, r, reduce8_src((lane - j0) & 7));
            if (lane >= j0 && lane < j0 + U) mine = got;
        }
        const int s = base + lane;
        if (s < k) {
            const bool ok = (okm >> lane) & 1u;
            double val = ok ? -g.scale * wd.w * mine : 0.0;
            if (bw.gd_acc) {
                if (f0 > 0) val += bw.gd_acc[v * k + s];
                if (!last_chunk) bw.gd_acc[v * k + s] = val;
            }
            if (last_chunk) bw.grad_d2[v * k + s] = (float)val;
        }
    }
}

// Single-gather row pass for k <= 64 (2 slot windows): the mean-block dot
// products and the running arg-max (value, slot, feature value at the max)
// come out of ONE gather sweep; the max blocks' share of grad_d2 (a few
// slots per row) is added through shared-memory float64 atomics afterwards,
// and their feature gradient goes to the arg-max neighbour as before.  Same
// arithmetic as k_gn_rows (which gathers twice: arg-max first, then the dots).
template <int VW>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_rows1(const GnArgs g, const GnBwd bw, int f0,
                                                           int last_chunk) {
    constexpr int UR = 4;  // gathers in flight (fewer registers, more warps)
    __shared__ double extra_s[kRowWarps][64];
    const int lane = lane_id();
    const int wi = threadIdx.x >> 5;
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + wi;
    if (p >= g.n) return;
    const int64_t v = row_of(g, p);
    const int k = g.k, F = g.F, W = F * g.n_red;
    const int fl = f0 + lane * VW;
    const bool lane_on = fl < F;
    const bool has_max = g.max_bits != 0;
    Window wd[2];
    int cnt = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        wd[h] = load_window(g, v, 32 * h, true);
        cnt += __popc(wd[h].okm);
        if (f0 == 0 && ((wd[h].okm >> lane) & 1u)) atomicAdd(&bw.rev_cnt[wd[h].u], 1);
    }
    extra_s[wi][lane] = 0.0;
    extra_s[wi][lane + 32] = 0.0;
    double cmean[VW], cmax[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        cmean[e] = 0.0;
        cmax[e] = 0.0;
    }
    if (lane_on && cnt > 0) {
        for (int b = 0; b < g.n_red; ++b) {
            float ub[VW];
            ldf<VW>(bw.up + v * W + (int64_t)b * F + fl, ub);
#pragma unroll
            for (int e = 0; e < VW; ++e) {
                if (is_max(g, b))
                    cmax[e] += (double)ub[e];
                else
                    cmean[e] += (double)ub[e] / (double)cnt;
            }
        }
    }
    if (lane_on && bw.has_mean) {
        float o[VW];
#pragma unroll
        for (int e = 0; e < VW; ++e) o[e] = (float)cmean[e];
        stf<VW>(bw.cm + v * F + fl, o);
    }
    double best[VW];
    int bslot[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) {
        best[e] = -INFINITY;
        bslot[e] = -1;
    }
    double mine[2] = {0.0, 0.0};  // this lane's slot: mean-block dot product
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const unsigned okm = cnt > 0 ? wd[h].okm : 0u;
        for (int j0 = 0; j0 < 32; j0 += UR) {
            if (((okm >> j0) & ((1u << UR) - 1u)) == 0) continue;
            float x[UR][VW];
            double w[UR];
            bool valid[UR];
            gather<VW, UR>(g, wd[h], j0, fl, lane_on, x, w, valid);
            double part[UR];
#pragma unroll
            for (int q = 0; q < UR; ++q) {
                part[q] = 0.0;
#pragma unroll
                for (int e = 0; e < VW; ++e) {
                    part[q] += (double)x[q][e] * cmean[e];
                    if (has_max && valid[q]) {
                        const double term = w[q] * (double)x[q][e];
                        if (term > best[e]) {
                            best[e] = term;
                            bslot[e] = 32 * h + j0 + q;
                        }
                    }
                }
            }
            const double r = transpose_reduce4(part);
            const double got = __shfl_sync(FG_FULL_MASK, r, reduce4_src((lane - j0) & 3));
            if (lane >= j0 && lane < j0 + UR) mine[h] = got;
        }
    }
    __syncwarp();
    // max blocks: slot bslot gets -scale w x cmax in grad_d2, neighbour u gets w cmax
    // (w and x at the arg-max are re-read: L1 hits, no per-element bookkeeping)
    if (has_max && lane_on && cnt > 0) {
#pragma unroll
        for (int e = 0; e < VW; ++e) {
            if (bslot[e] < 0) continue;
            const int32_t u = __ldg(&g.idx[v * k + bslot[e]]);
            const double wb = exp(-g.scale * (double)__ldg(&g.d2[v * k + bslot[e]]));
            const float xb = __ldg(&g.feats[(int64_t)u * F + fl + e]);
            atomicAdd(&extra_s[wi][bslot[e]], (double)xb * cmax[e]);
#ifndef FG_GN_NO_GMAX  // timing experiment only
            if (bw.gmax) atomicAdd(&bw.gmax[(int64_t)u * F + fl + e], wb * cmax[e]);
#endif
        }
    }
    __syncwarp();
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int s = 32 * h + lane;
        if (s < k) {
            const bool ok = cnt > 0 && ((wd[h].okm >> lane) & 1u);
            double val = ok ? -g.scale * wd[h].w * (mine[h] + extra_s[wi][s]) : 0.0;
            if (bw.gd_acc) {
                if (f0 > 0) val += bw.gd_acc[v * k + s];
                if (!last_chunk) bw.gd_acc[v * k + s] = val;
            }
            if (last_chunk) bw.grad_d2[v * k + s] = (float)val;
        }
    }
}

// Reverse fill: entry v*k + s goes to neighbour u's list.
__global__ void k_gn_fill(const GnArgs g, const GnBwd bw) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= g.n * g.k) return;
    const int64_t v = t / g.k;
    const int s = (int)(t - v * g.k);
    const int32_t u = g.idx[t];
    if (!slot_valid(g, s, u)) return;
    bw.rev[atomicAdd(&bw.rev_cur[u], 1)] = (int32_t)t;
}

// Column pass: grad_feats[u] = sum over u's reverse list of w_vs cm[v] (+ the
// max-block gradient scattered to u), float64.  The sum over the list is
// order-independent up to float64 rounding (the list order comes from the
// atomic fill), far inside the float32 output precision.
#ifndef FG_GN_COLS_U
#define FG_GN_COLS_U 2
#endif
template <int VW>
__global__ void __launch_bounds__(kRowWarps * 32) k_gn_cols(const GnArgs g, const GnBwd bw, int f0) {
    constexpr int UC = FG_GN_COLS_U;
    const int lane = lane_id();
    const int64_t p = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (p >= g.n) return;
    const int64_t u = row_of(g, p);
    const int k = g.k, F = g.F;
    const int fl = f0 + lane * VW;
    const bool lane_on = fl < F;
    double acc[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) acc[e] = 0.0;
    if (bw.has_mean) {
        const int32_t lo = bw.rev_off[u], hi = bw.rev_off[u + 1];
        for (int32_t base = lo; base < hi; base += 32) {
            const int32_t ent = base + lane;
            int32_t vv = 0;
            double w = 0.0;
            if (ent < hi) {
                const int32_t t = bw.rev[ent];
                vv = t / k;
                w = exp(-g.scale * (double)__ldg(&g.d2[t]));
            }
            const int nb = min(32, hi - base);
            for (int j0 = 0; j0 < nb; j0 += UC) {
                float x[UC][VW];
                double wq[UC];
#pragma unroll
                for (int q = 0; q < UC; ++q) {
                    const int32_t vq = __shfl_sync(FG_FULL_MASK, vv, (j0 + q) & 31);
                    wq[q] = __shfl_sync(FG_FULL_MASK, w, (j0 + q) & 31);
#pragma unroll
                    for (int e = 0; e < VW; ++e) x[q][e] = 0.0f;
                    if (j0 + q < nb && lane_on) ldf<VW>(bw.cm + (int64_t)vq * F + fl, x[q]);
                }
#pragma unroll
                for (int q = 0; q < UC; ++q) {
#pragma unroll
                    for (int e = 0; e < VW; ++e) acc[e] += wq[q] * (double)x[q][e];
                }
            }
        }
    }
    if (!lane_on) return;
    if (bw.gmax) {
#pragma unroll
        for (int e = 0; e < VW; ++e) acc[e] += bw.gmax[u * F + fl + e];
    }
    float o[VW];
#pragma unroll
    for (int e = 0; e < VW; ++e) o[e] = (float)acc[e];
    stf<VW>(bw.grad_feats + u * F + fl, o);
}

int check_reducers(const int32_t* reducers, int32_t n_red, GnArgs& g) {
    if (!reducers) return FG_ERR_NULL;
    if (n_red < 1 || n_red > 4) return FG_ERR_BAD_SHAPE;
    g.max_bits = 0;
    for (int i = 0; i < n_red; ++i) {
        if (reducers[i] != FG_REDUCE_MEAN && reducers[i] != FG_REDUCE_MAX) return FG_ERR_BAD_SHAPE;
        if (reducers[i] == FG_REDUCE_MAX) g.max_bits |= 1u << i;
    }
    g.n_red = n_red;
    return 0;
}

// Features per lane: float4 / float2 loads when the row length and every
// feature-row base pointer allow it.
int pick_vw(int F, std::initializer_list<const void*> ptrs) {
    auto aligned = [&](size_t a) {
        for (const void* p : ptrs)
            if (p && ((uintptr_t)p % a) != 0) return false;
        return true;
    };
    if (F % 4 == 0 && F > 64 && aligned(16)) return 4;
    if (F % 2 == 0 && F > 32 && aligned(8)) return 2;
    return 1;
}

template <typename Launch>
int with_vw(int vw, Launch&& launch) {
    if (vw == 4) return launch(std::integral_constant<int, 4>{});
    if (vw == 2) return launch(std::integral_constant<int, 2>{});
    return launch(std::integral_constant<int, 1>{});
}

struct BwdWs {
    float* cm;
    double* gmax;
    double* gd_acc;
    int32_t* rev_cnt;
    int32_t* rev_off;
    int32_t* rev_cur;
    int32_t* rev;
    unsigned long long* status;
    unsigned* ticket;
    int64_t n_tiles;
};

// gd_acc is sized for the worst case (one-wide lanes: 32 features per chunk).
size_t carve(BwdWs* w, void* base, int64_t n, int F, int k) {
    size_t off = 0;
    char* b = (char*)base;
    auto take = [&](size_t bytes) {
        off = align_up(off, 256);
        char* p = b ? b + off : nullptr;
        off += bytes;
        return p;
    };
    w->n_tiles = ceil_div(n, kScanTile);
    w->cm = (float*)take(sizeof(float) * (size_t)n * F);
    w->gmax = (double*)take(sizeof(double) * (size_t)n * F);
    w->gd_acc = F > 32 ? (double*)take(sizeof(double) * (size_t)n * k) : nullptr;
    w->rev_cnt = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w->rev_off = (int32_t*)take(sizeof(int32_t) * (size_t)(n + 1));
    w->rev_cur = (int32_t*)take(sizeof(int32_t) * (size_t)n);
    w->rev = (int32_t*)take(sizeof(int32_t) * (size_t)n * k);
    w->status = (unsigned long long*)take(sizeof(unsigned long long) * (size_t)(w->n_tiles + 1));
    w->ticket = (unsigned*)take(sizeof(unsigned) * 4);
    return align_up(off, 256);
}

template <int VW>
int gn_backward(const GnArgs& g, GnBwd bw, const BwdWs& w, cudaStream_t st) {
    constexpr int CW = 32 * VW;
    if (g.F <= CW) bw.gd_acc = nullptr;
    const unsigned blocks = (unsigned)ceil_div(g.n, kRowWarps);
    for (int f0 = 0; f0 < g.F; f0 += CW) {
        if (g.k <= 64)
            k_gn_rows1<VW><<<blocks, kRowWarps * 32, 0, st>>>(g, bw, f0, f0 + CW >= g.F);
        else
            k_gn_rows<VW><<<blocks, kRowWarps * 32, 0, st>>>(g, bw, f0, f0 + CW >= g.F);
        FG_TRY(launched(st));
    }
    if (bw.has_mean) {
        k_scan<<<(unsigned)w.n_tiles, kScanThreads, 0, st>>>(w.rev_cnt, g.n, w.rev_off, w.rev_cur,
                                                            w.status, w.ticket);
        FG_TRY(launched(st));
        k_gn_fill<<<(unsigned)ceil_div(g.n * g.k, 256), 256, 0, st>>>(g, bw);
        FG_TRY(launched(st));
    }
    for (int f0 = 0; f0 < g.F; f0 += CW) {
        k_gn_cols<VW><<<blocks, kRowWarps * 32, 0, st>>>(g, bw, f0);
        FG_TRY(launched(st));
    }
    return 0;
}

int reducer_bits(const int32_t* reducers, int n_red, unsigned* bits) {
    GnArgs g;
    FG_TRY(check_reducers(reducers, n_red, g));
    *bits = g.max_bits;
    return 0;
}

}  // namespace gravnet
}  // namespace fg

using namespace fg;
using namespace fg::gravnet;

extern "C" int fg_gravnet_fwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              const int32_t* order, float* out, void* stream) {
    GnArgs g;
    FG_TRY(check_reducers(reducers, n_reducers, g));
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !out) return FG_ERR_NULL;
    g.feats = feats; g.n = n; g.F = n_feats; g.idx = idx; g.d2 = d2; g.k = k;
    g.scale = weight_scale; g.include_self = include_self; g.order = order;
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)ceil_div(n, kRowWarps);
    if (n_feats % 4 == 0 && n_feats <= 64 && ((uintptr_t)feats % 16) == 0 && ((uintptr_t)out % 16) == 0) {
        k_gn_fwd_pairs<FG_GN_PAIRS_U><<<blocks, kRowWarps * 32, 0, st>>>(g, out);
        return launched(st);
    }
    return with_vw(pick_vw(n_feats, {feats, out}), [&](auto vw) {
        constexpr int VW = decltype(vw)::value;
        for (int f0 = 0; f0 < n_feats; f0 += 32 * VW) {
            k_gn_fwd<VW><<<blocks, kRowWarps * 32, 0, st>>>(g, f0, out);
            FG_TRY(launched(st));
        }
        return 0;
    });
}

extern "C" int fg_gravnet_bwd_workspace_size(int64_t n, int32_t n_feats, int32_t k, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    BwdWs w;
    *bytes = carve(&w, nullptr, n, n_feats, k);
    return 0;
}

extern "C" int fg_gravnet_bwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              const int32_t* order, const float* upstream, float* grad_feats,
                              float* grad_d2, void* workspace, size_t workspace_bytes,
                              void* stream) {
    GnArgs g;
    FG_TRY(check_reducers(reducers, n_reducers, g));
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if ((int64_t)n * k >= (int64_t)INT32_MAX) return FG_ERR_BAD_SHAPE;  // 32-bit reverse entries
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !upstream || !grad_feats || !grad_d2 || !workspace) return FG_ERR_NULL;
    BwdWs w;
    const size_t need = carve(&w, workspace, n, n_feats, k);
    if (workspace_bytes < need) return FG_ERR_WORKSPACE;
    g.feats = feats; g.n = n; g.F = n_feats; g.idx = idx; g.d2 = d2; g.k = k;
    g.scale = weight_scale; g.include_self = include_self; g.order = order;
    const unsigned all_bits = (1u << g.n_red) - 1u;
    GnBwd bw;
    bw.up = upstream; bw.cm = w.cm; bw.gmax = g.max_bits ? w.gmax : nullptr; bw.grad_d2 = grad_d2;
    bw.gd_acc = w.gd_acc; bw.rev_cnt = w.rev_cnt; bw.rev_off = w.rev_off; bw.rev_cur = w.rev_cur;
    bw.rev = w.rev; bw.grad_feats = grad_feats; bw.has_mean = g.max_bits != all_bits;
    cudaStream_t st = (cudaStream_t)stream;
    FG_CUDA(cudaMemsetAsync(w.rev_cnt, 0, sizeof(int32_t) * (size_t)n, st));
    FG_CUDA(cudaMemsetAsync(w.status, 0, sizeof(unsigned long long) * (size_t)(w.n_tiles + 1), st));
    FG_CUDA(cudaMemsetAsync(w.ticket, 0, sizeof(unsigned) * 4, st));
    if (bw.gmax) FG_CUDA(cudaMemsetAsync(bw.gmax, 0, sizeof(double) * (size_t)n * n_feats, st));
    return with_vw(pick_vw(n_feats, {feats, upstream, grad_feats}), [&](auto vw) {
        constexpr int VW = decltype(vw)::value;
        return gn_backward<VW>(g, bw, w, st);
    });
}
