// fg_grad.cu -- binned_select_knn backward (replaces G/knn.py:135-168) for
// sm_100a.
//
// Precision: every knn_backward term 2g(x_v - x_u) is formed exactly in float64
// (fp32 g and x), the query-side sum of a row is a warp reduction in float64,
// and both sides reach the per-vertex accumulator through compensated fp32x4
// atomics (hi + exact-TwoSum error, see two_sum_add): ~2^-48 relative to the
// term magnitudes, i.e. float64-class, then rounded once to the output type.
#include "fg_common.cuh"

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
        lp[i] = (float)(x[i] - (double)hp[i]);
    }
    const float4 old = atomicAdd(hi_acc, h);
    const float* op = &old.x;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const float a = op[i], b = hp[i];
        const float sum = __fadd_rn(a, b);
        const float bb = __fsub_rn(sum, a);
        const float err = __fadd_rn(__fsub_rn(a, __fsub_rn(sum, bb)), __fsub_rn(b, bb));
        lp[i] = __fadd_rn(lp[i], err);
    }
    atomicAdd(lo_acc, l);
}

// Warp per row (visited in `order` when given: spatially sorted rows keep the
// neighbour gathers and the atomic targets local), lanes over slots.
template <int NV>
__global__ void __launch_bounds__(kRowWarps * 32) k_knn_bwd(const float* __restrict__ coords, int64_t n,
                                                          int n_c, const int32_t* __restrict__ idx,
                                                          int k, const float* __restrict__ gd2,
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
                    c[e] = two_g * (xv[i] - xu);  // exact: 24-bit g times a 25-bit difference
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

// d <= 4, k <= 65: RPW rows per warp with every (row, slot-round) chain in
// flight at once -- the coordinate gathers, then the returning fp32x4 atomics,
// then the TwoSum corrections -- so the L2 round trips of 2*RPW chains overlap
// (the warp-per-row kernel above waits for each one).  Same arithmetic.
#ifndef FG_BWD_MINB
#define FG_BWD_MINB 4
#endif
template <int RPW, int SR>
__global__ void __launch_bounds__(kRowWarps * 32, FG_BWD_MINB) k_knn_bwd_pipe(
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
            lp[i] = __fadd_rn(lp[i], err);
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

__global__ void k_bwd_finish(const float4* __restrict__ hi, const float4* __restrict__ lo, int64_t n,
                             int n_c, int nv, void* __restrict__ out, int is_f64) {
    const int64_t m = n * n_c;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t v = t / n_c;
        const int i = (int)(t - v * n_c);
        const float h = (&hi[v * nv + (i >> 2)].x)[i & 3];
        const float l = (&lo[v * nv + (i >> 2)].x)[i & 3];
        const double x = (double)h + (double)l;
        if (is_f64)
            reinterpret_cast<double*>(out)[t] = x;
        else
            reinterpret_cast<float*>(out)[t] = (float)x;
    }
}

}  // namespace grad
}  // namespace fg

using namespace fg;
using namespace fg::grad;

extern "C" int fg_knn_bwd_workspace_size(int64_t n, int32_t n_coords, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_coords < 1) return FG_ERR_BAD_SHAPE;
    const int nv = (n_coords + 3) / 4;
    *bytes = 2 * align_up(sizeof(float4) * (size_t)n * nv, 256);
    return 0;
}

extern "C" int fg_knn_bwd(const float* coords, int64_t n, int32_t n_coords, const int32_t* idx,
                          int32_t k, const float* grad_d2, const int32_t* order, void* grad_coords,
                          int32_t grad_is_f64, void* workspace, size_t workspace_bytes,
                          void* stream) {
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_coords < 1) return FG_ERR_BAD_SHAPE;
    if (n_coords > 16) return FG_ERR_TOO_MANY_DIMS;
    if (n == 0) return 0;
    if (!coords || !idx || !grad_d2 || !grad_coords || !workspace) return FG_ERR_NULL;
    const int nv = (n_coords + 3) / 4;
    const size_t half = align_up(sizeof(float4) * (size_t)n * nv, 256);
    if (workspace_bytes < 2 * half) return FG_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    float4* hi = (float4*)workspace;
    float4* lo = (float4*)((char*)workspace + half);
    FG_CUDA(cudaMemsetAsync(workspace, 0, 2 * half, st));
    const unsigned blocks = (unsigned)ceil_div(n, kRowWarps);
#ifndef FG_BWD_RPW
#define FG_BWD_RPW 1
#endif
    constexpr int RPW = FG_BWD_RPW;
    const unsigned pblocks = (unsigned)ceil_div(n, (int64_t)kRowWarps * RPW);
    if (nv == 1 && k <= 33) {
        k_knn_bwd_pipe<RPW, 1><<<pblocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo);
    } else if (nv == 1 && k <= 65) {
        k_knn_bwd_pipe<RPW, 2><<<pblocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo);
    } else switch (nv) {
        case 1: k_knn_bwd<1><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        case 2: k_knn_bwd<2><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        case 3: k_knn_bwd<3><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
        default: k_knn_bwd<4><<<blocks, kRowWarps * 32, 0, st>>>(coords, n, n_coords, idx, k, grad_d2, order, hi, lo); break;
    }
    FG_TRY(launched(st));
    const int64_t m = n * n_coords;
    k_bwd_finish<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 148 * 16), 256, 0, st>>>(
        hi, lo, n, n_coords, nv, grad_coords, grad_is_f64);
    return launched(st);
}
