// fg_common.cuh -- shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/fastgraph_b200.h"

#define FG_FULL_MASK 0xffffffffu

namespace fg {

// Number of kernels launched through this library (fg_launch_count()).
extern std::atomic<uint64_t> g_launches;

inline int launched(cudaStream_t) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? 0 : (int)e;
}

#define FG_TRY(expr)                 \
    do {                             \
        int _rc = (expr);            \
        if (_rc != 0) return _rc;    \
    } while (0)

#define FG_CUDA(expr)                         \
    do {                                      \
        cudaError_t _e = (expr);              \
        if (_e != cudaSuccess) return (int)_e; \
    } while (0)

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Order-preserving float <-> uint32 map (all finite floats, +-inf).
__device__ __forceinline__ unsigned float_to_ordered(float f) {
    unsigned b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(unsigned u) {
    unsigned b = (u & 0x80000000u) ? (u & 0x7fffffffu) : ~u;
    return __uint_as_float(b);
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T t = __shfl_up_sync(FG_FULL_MASK, v, o);
        if (lane_id() >= o) v += t;
    }
    return v;
}

// Exact float64 squared distance in the reference's operation order
// (_binned_cy.pyx:32-48: acc = (a0-b0)^2, acc = acc + (ai-bi)^2 ...),
// explicit _rn intrinsics so nothing is contracted into an FMA.
template <int NC_MAX>
__device__ __forceinline__ double exact_d2(const float* q, const float* c, int n_c) {
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < NC_MAX; ++i) {
        if (i < n_c) {
            double t = __dsub_rn((double)q[i], (double)c[i]);
            double sq = __dmul_rn(t, t);
            acc = (i == 0) ? sq : __dadd_rn(acc, sq);
        }
    }
    return acc;
}

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

__host__ __device__ inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Split of vertex v: the unique s with rs[s] <= v < rs[s+1] (bisect-right - 1,
// _binned_cy.pyx:51-60); empty splits are skipped naturally.
__device__ __forceinline__ int split_of(const int64_t* rs, int n_splits, int64_t v) {
    int lo = 0, hi = n_splits + 1;
    while (lo < hi) {
        int mid = (lo + hi) >> 1;
        if (rs[mid] <= v)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo - 1;
}

}  // namespace fg
