// Microbenchmark: scattered 32-byte float64x4 additions to 1M accumulators by
// TMA bulk reductions (cp.reduce.async.bulk .add.f64 from shared memory), vs the
// backward's current pair (returning float4 ATOM + float4 RED), 40M terms each.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
// MODE 0: bulk f64 reduce, one 32-byte op per term, issued by every lane
// MODE 1: float4 ATOM (returning) + float4 RED per term (the current backward)
// MODE 2: bulk f64 reduce, 4 terms staged per lane before one commit/wait
template <int MODE>
__global__ void __launch_bounds__(256) k(double* acc64, float* acc32, int64_t nops, uint32_t nslots, float* sink) {
  __shared__ __align__(16) double st[256][4 * 4];
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float a = 0.f;
  if (MODE == 0) {
    for (int64_t i = t; i < nops; i += stride) {
      uint32_t s = hash32((uint32_t)i) % nslots;
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      st[threadIdx.x][0] = 1.0; st[threadIdx.x][1] = 2.0; st[threadIdx.x][2] = 3.0; st[threadIdx.x][3] = (double)i;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint32_t src = (uint32_t)__cvta_generic_to_shared(&st[threadIdx.x][0]);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 32;"
                   :: "l"(acc64 + 4 * (size_t)s), "r"(src) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (MODE == 2) {
    int slot = 0;
    for (int64_t i = t; i < nops; i += stride) {
      uint32_t s = hash32((uint32_t)i) % nslots;
      if (slot == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      double* p = &st[threadIdx.x][4 * slot];
      p[0] = 1.0; p[1] = 2.0; p[2] = 3.0; p[3] = (double)i;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      uint32_t src = (uint32_t)__cvta_generic_to_shared(p);
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], 32;"
                   :: "l"(acc64 + 4 * (size_t)s), "r"(src) : "memory");
      if (++slot == 4) { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); slot = 0; }
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  if (MODE == 1) {
    for (int64_t i = t; i < nops; i += stride) {
      uint32_t s = hash32((uint32_t)i) % nslots;
      float4 o = atomicAdd(reinterpret_cast<float4*>(acc32) + s, make_float4(1.f, 2.f, 3.f, 4.f));
      atomicAdd(reinterpret_cast<float4*>(acc32) + nslots + s, make_float4(o.x * 1e-8f, 0.f, 0.f, 0.f));
    }
  }
  if (a == 12345.f) sink[0] = a;
}
template <int MODE> float run(double* a64, float* a32, int64_t nops, uint32_t nslots, float* sink) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 8, 256>>>(a64, a32, nops, nslots, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE><<<148 * 8, 256>>>(a64, a32, nops, nslots, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
  double* a64; float* a32; float* sink;
  cudaMalloc(&a64, 1000000 * 32); cudaMalloc(&a32, 1000000 * 32); cudaMalloc(&sink, 4096 * 4);
  cudaMemset(a64, 0, 1000000 * 32); cudaMemset(a32, 0, 1000000 * 32);
  const int64_t n = 40000000;
  printf("bulk f64x4 reduce, 1 per group   %.3f ms\n", run<0>(a64, a32, n, 1000000, sink));
  printf("bulk f64x4 reduce, 4 per group   %.3f ms\n", run<2>(a64, a32, n, 1000000, sink));
  printf("float4 ATOM + float4 RED         %.3f ms\n", run<1>(a64, a32, n, 1000000, sink));
  double h[4];
  cudaMemcpy(h, a64, 32, cudaMemcpyDeviceToHost);
  printf("check slot0: %.1f %.1f %.1f\n", h[0], h[1], h[2]);
  return 0;
}
