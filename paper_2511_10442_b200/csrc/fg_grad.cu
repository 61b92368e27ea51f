// fg_grad.cu -- binned_select_knn backward (replaces G/knn.py:135-168) and the
// GravNet distance-weighted aggregation forward/backward (replaces
// G/gravnet.py:64-150) for sm_100a.
//
// Precision: every knn_backward term 2g(x_v - x_u) is formed exactly in float64
// (fp32 g and x), the query-side sum of a row is a warp reduction in float64,
// and both sides reach the per-vertex accumulator through compensated fp32x4
// atomics (hi + exact-TwoSum error, see two_sum_add): ~2^-48 relative to the
// term magnitudes, i.e. float64-class, then rounded once to the output type.  GravNet weights exp(-scale d2), the
// weighted terms, sums and maxima are float64 and stored
// as float32.
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

__global__ void k_round_out(const double* __restrict__ acc, int64_t m, void* __restrict__ out, int is_f64) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (is_f64)
            reinterpret_cast<double*>(out)[i] = acc[i];
        else
            reinterpret_cast<float*>(out)[i] = (float)acc[i];
    }
}

// ---------------------------------------------------------------- GravNet
// Warp per vertex; lanes over features (FPL features per lane per pass).
__global__ void __launch_bounds__(kRowWarps * 32) k_gravnet_fwd(const float* __restrict__ feats, int64_t n,
                                                              int F, const int32_t* __restrict__ idx,
                                                              const float* __restrict__ d2, int k,
                                                              double scale, int4 red, int n_red,
                                                              int include_self, float* __restrict__ out) {
    const int lane = lane_id();
    const int64_t v = blockIdx.x * (int64_t)kRowWarps + (threadIdx.x >> 5);
    if (v >= n) return;
    const int W = F * n_red;
    int cnt = 0;
    for (int base = 0; base < k; base += 32) {
        const int s = base + lane;
        const bool ok = s < k && idx[v * k + s] >= 0 && (include_self || s > 0);
        cnt += __popc(__ballot_sync(FG_FULL_MASK, ok));
    }
    const int reds[4] = {red.x, red.y, red.z, red.w};
    for (int f0 = 0; f0 < F; f0 += 32) {
        const int f = f0 + lane;
        double sum = 0.0, mx = -INFINITY;
        for (int base = 0; base < k; base += 32) {
            const int s = base + lane;
            int32_t u = s < k ? idx[v * k + s] : -1;
            const bool ok = u >= 0 && (include_self || s > 0);
            const double w = ok ? exp(-scale * (double)d2[v * k + s]) : 0.0;
            const unsigned okm = __ballot_sync(FG_FULL_MASK, ok);
            const int lim = min(32, k - base);
            for (int j = 0; j < lim; ++j) {
                if (!((okm >> j) & 1u)) continue;
                const int32_t uj = __shfl_sync(FG_FULL_MASK, u, j);
                const double wj = __shfl_sync(FG_FULL_MASK, w, j);
                if (f < F) {
                    const double term = wj * (double)feats[(int64_t)uj * F + f];
                    sum += term;
                    if (term > mx) mx = term;
                }
            }
        }
        if (f < F) {
            for (int b = 0; b < n_red; ++b) {
                double val = 0.0;
                if (cnt > 0) val = reds[b] == FG_REDUCE_MEAN ? sum / (double)cnt : mx;
                out[v * W + (int64_t)b * F + f] = (float)val;
            }
        }
    }
}

// grad_feats via float64 atomics into gacc[n*F]; grad_d2 per row in smem.
__global__ void __launch_bounds__(kRowWarps * 32) k_gravnet_bwd(const float* __restrict__ feats, int64_t n,
                                                              int F, const int32_t* __restrict__ idx,
                                                              const float* __restrict__ d2, int k,
                                                              double scale, int4 red, int n_red,
                                                              int include_self,
                                                              const float* __restrict__ up,
                                                              double* __restrict__ gacc,
                                                              float* __restrict__ grad_d2) {
    extern __shared__ double s_gd[];
    const int lane = lane_id();
    const int wib = threadIdx.x >> 5;
    double* gd = s_gd + (size_t)wib * k;
    const int64_t v = blockIdx.x * (int64_t)kRowWarps + wib;
    if (v >= n) return;
    const int W = F * n_red;
    for (int s = lane; s < k; s += 32) gd[s] = 0.0;
    int cnt = 0;
    for (int base = 0; base < k; base += 32) {
        const int s = base + lane;
        const bool ok = s < k && idx[v * k + s] >= 0 && (include_self || s > 0);
        cnt += __popc(__ballot_sync(FG_FULL_MASK, ok));
    }
    __syncwarp();
    const int reds[4] = {red.x, red.y, red.z, red.w};
    if (cnt > 0) {
        for (int b = 0; b < n_red; ++b) {
            const bool is_mean = reds[b] == FG_REDUCE_MEAN;
            for (int f0 = 0; f0 < F; f0 += 32) {
                const int f = f0 + lane;
                const double g = f < F ? (double)up[v * W + (int64_t)b * F + f] : 0.0;
                const double coeff = g / (double)cnt;
                double best = -INFINITY;
                int best_s = -1;
                int32_t best_u = 0;
                double best_w = 0.0;
                for (int base = 0; base < k; base += 32) {
                    const int s = base + lane;
                    const int32_t u = s < k ? idx[v * k + s] : -1;
                    const bool ok = u >= 0 && (include_self || s > 0);
                    const double w = ok ? exp(-scale * (double)d2[v * k + s]) : 0.0;
                    const unsigned okm = __ballot_sync(FG_FULL_MASK, ok);
                    const int lim = min(32, k - base);
                    for (int j = 0; j < lim; ++j) {
                        if (!((okm >> j) & 1u)) continue;
                        const int32_t uj = __shfl_sync(FG_FULL_MASK, u, j);
                        const double wj = __shfl_sync(FG_FULL_MASK, w, j);
                        const double fv = f < F ? (double)feats[(int64_t)uj * F + f] : 0.0;
                        if (is_mean) {
                            if (f < F) atomicAdd(&gacc[(int64_t)uj * F + f], wj * coeff);
                            double dot = fv * coeff;
#pragma unroll
                            for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(FG_FULL_MASK, dot, o);
                            if (lane == 0) gd[base + j] += -scale * wj * dot;
                        } else {
                            const double term = wj * fv;
                            if (f < F && term > best) {
                                best = term;
                                best_s = base + j;
                                best_u = uj;
                                best_w = wj;
                            }
                        }
                    }
                    __syncwarp();
                }
                if (!is_mean && f < F && best_s >= 0) {
                    atomicAdd(&gacc[(int64_t)best_u * F + f], g * best_w);
                    atomicAdd(&gd[best_s], ((-scale * g) * best_w) * (double)feats[(int64_t)best_u * F + f]);
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    for (int s = lane; s < k; s += 32) grad_d2[v * k + s] = (float)gd[s];
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
    switch (nv) {
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

static int check_reducers(const int32_t* reducers, int32_t n_red, int4* red) {
    if (!reducers) return FG_ERR_NULL;
    if (n_red < 1 || n_red > 4) return FG_ERR_BAD_SHAPE;
    int r[4] = {0, 0, 0, 0};
    for (int i = 0; i < n_red; ++i) {
        if (reducers[i] != FG_REDUCE_MEAN && reducers[i] != FG_REDUCE_MAX) return FG_ERR_BAD_SHAPE;
        r[i] = reducers[i];
    }
    *red = make_int4(r[0], r[1], r[2], r[3]);
    return 0;
}

extern "C" int fg_gravnet_fwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              float* out, void* stream) {
    int4 red;
    FG_TRY(check_reducers(reducers, n_reducers, &red));
    if (k < 1) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !out) return FG_ERR_NULL;
    cudaStream_t st = (cudaStream_t)stream;
    k_gravnet_fwd<<<(unsigned)ceil_div(n, kRowWarps), kRowWarps * 32, 0, st>>>(
        feats, n, n_feats, idx, d2, k, weight_scale, red, n_reducers, include_self, out);
    return launched(st);
}

extern "C" int fg_gravnet_bwd_workspace_size(int64_t n, int32_t n_feats, size_t* bytes) {
    if (!bytes) return FG_ERR_NULL;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    *bytes = align_up(sizeof(double) * (size_t)n * n_feats, 256);
    return 0;
}

extern "C" int fg_gravnet_bwd(const float* feats, int64_t n, int32_t n_feats, const int32_t* idx,
                              const float* d2, int32_t k, double weight_scale,
                              const int32_t* reducers, int32_t n_reducers, int32_t include_self,
                              const float* upstream, float* grad_feats, float* grad_d2,
                              void* workspace, size_t workspace_bytes, void* stream) {
    int4 red;
    FG_TRY(check_reducers(reducers, n_reducers, &red));
    if (k < 1 || k > 4096) return FG_ERR_BAD_K;
    if (n < 0 || n_feats < 1) return FG_ERR_BAD_SHAPE;
    if (!(weight_scale > 0.0)) return FG_ERR_BAD_SHAPE;
    if (n == 0) return 0;
    if (!feats || !idx || !d2 || !upstream || !grad_feats || !grad_d2 || !workspace) return FG_ERR_NULL;
    const size_t need = align_up(sizeof(double) * (size_t)n * n_feats, 256);
    if (workspace_bytes < need) return FG_ERR_WORKSPACE;
    cudaStream_t st = (cudaStream_t)stream;
    double* gacc = (double*)workspace;
    FG_CUDA(cudaMemsetAsync(gacc, 0, sizeof(double) * (size_t)n * n_feats, st));
    const size_t smem = sizeof(double) * (size_t)k * kRowWarps;
    if (smem > 48 * 1024)
        FG_CUDA(cudaFuncSetAttribute(k_gravnet_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gravnet_bwd<<<(unsigned)ceil_div(n, kRowWarps), kRowWarps * 32, smem, st>>>(
        feats, n, n_feats, idx, d2, k, weight_scale, red, n_reducers, include_self, upstream, gacc,
        grad_d2);
    FG_TRY(launched(st));
    const int64_t m = n * n_feats;
    k_round_out<<<(unsigned)std::min<int64_t>(ceil_div(m, 256), 148 * 8), 256, 0, st>>>(gacc, m, grad_feats, 0);
    return launched(st);
}
