// Experiment: knn backward with accumulators indexed by SORTED POSITION and the
// neighbour slots of a row visited in ascending position order, so that
// neighbouring lanes hit neighbouring 16-byte accumulator slots (the locality
// microbenchmark red_locality.cu: 2-8 lanes per sector ~2x the RED/ATOM rate).
// variant 0: posmat rows as given; variant 1: the kernel sorts each 32-slot
// round by position with a warp bitonic sort first.  Built as a small .so and
// driven by tools/bwd_pos.py (timing only; the arithmetic is the product's).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

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
        lp[i] = __fadd_rn(lp[i], __fadd_rn(__fsub_rn(a, __fsub_rn(sum, bb)), __fsub_rn(b, bb)));
    }
    atomicAdd(lo_acc, l);
}

__device__ __forceinline__ unsigned bitonic32(unsigned key) {
    const int lane = lane_id();
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            const unsigned o = __shfl_xor_sync(0xffffffffu, key, stride);
            const bool up = (lane & size) == 0;
            const bool lower = (lane & stride) == 0;
            const unsigned mn = min(key, o), mx = max(key, o);
            key = (lower == up) ? mn : mx;
        }
    }
    return key;
}

template <int SR, bool SORT>
__global__ void __launch_bounds__(256, 4) k_bwd_pos(const float4* __restrict__ sc, int64_t n, const int32_t* __restrict__ pm,
                                                   int k, const float* __restrict__ gm, float4* __restrict__ hi,
                                                   float4* __restrict__ lo) {
    const int lane = lane_id();
    const int64_t p = blockIdx.x * 8ll + (threadIdx.x >> 5);
    if (p >= n) return;
    const float4 a = sc[p];
    double qs[4] = {0, 0, 0, 0};
#pragma unroll
    for (int q = 0; q < SR; ++q) {
        const int s = 1 + lane + 32 * q;
        int32_t u = s < k ? pm[p * k + s] : -1;
        float g = s < k ? gm[p * k + s] : 0.f;
        if (SORT) {  // (position << 6 | slot) sorted ascending; invalid last
            unsigned key = u >= 0 ? ((unsigned)u << 6) | (unsigned)(s & 63) : 0xffffffffu;
            key = bitonic32(key);
            const int src = key == 0xffffffffu ? lane : ((int)(key & 63) - 1 - 32 * q);
            g = __shfl_sync(0xffffffffu, g, src & 31);
            u = key == 0xffffffffu ? -1 : (int32_t)(key >> 6);
        }
        if (u >= 0) {
            const float4 b = sc[u];
            const double tg = 2.0 * (double)g;
            const double x[4] = {-(tg * ((double)a.x - (double)b.x)), -(tg * ((double)a.y - (double)b.y)),
                                 -(tg * ((double)a.z - (double)b.z)), -(tg * ((double)a.w - (double)b.w))};
            qs[0] -= x[0]; qs[1] -= x[1]; qs[2] -= x[2]; qs[3] -= x[3];
            two_sum_add(hi + u, lo + u, x);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) qs[i] += __shfl_xor_sync(0xffffffffu, qs[i], o);
    if (lane == 0) two_sum_add(hi + p, lo + p, qs);
}

extern "C" int bwd_pos(const void* sc, int64_t n, const int32_t* pm, int k, const float* gm, void* hi, void* lo,
                       int variant, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const unsigned blocks = (unsigned)((n + 7) / 8);
    if (variant == 1)
        k_bwd_pos<2, true><<<blocks, 256, 0, st>>>((const float4*)sc, n, pm, k, gm, (float4*)hi, (float4*)lo);
    else
        k_bwd_pos<2, false><<<blocks, 256, 0, st>>>((const float4*)sc, n, pm, k, gm, (float4*)hi, (float4*)lo);
    return (int)cudaGetLastError();
}
