// Microbenchmark: throughput of scattered global reductions on B200
// (scalar f32 / float4 / u64 / f64 RED, returning float4 ATOM) into an
// L2-resident array, 40M lane operations each.  Used to size the backward.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void k(float* a, int64_t nops, uint32_t nslots, float* sink) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  for (int64_t i = t; i < nops; i += stride) {
    uint32_t s = hash32((uint32_t)i) % nslots;
    if (MODE == 0) atomicAdd(a + s, 1.0f);
    if (MODE == 1) atomicAdd(reinterpret_cast<float4*>(a) + s, make_float4(1.f, 2.f, 3.f, 4.f));
    if (MODE == 2) atomicAdd(reinterpret_cast<unsigned long long*>(a) + s, 3ull);
    if (MODE == 3) atomicAdd(reinterpret_cast<double*>(a) + s, 1.0);
    if (MODE == 4) { float4 o = atomicAdd(reinterpret_cast<float4*>(a) + s, make_float4(1.f, 2.f, 3.f, 4.f)); acc += o.x; }
    if (MODE == 5) atomicAdd(reinterpret_cast<unsigned*>(a) + s, 1u);
    if (MODE == 6) { // float2 vector red
      atomicAdd(reinterpret_cast<float2*>(a) + s, make_float2(1.f, 2.f)); }
  }
  if (acc == 12345.f) sink[0] = acc;
}
template <int MODE>
__global__ void ks(float* out, int64_t nops_per_block) {  // shared-memory atomics
  __shared__ uint32_t h[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < nops_per_block; i += blockDim.x) {
    uint32_t s = hash32((uint32_t)(i + blockIdx.x * 77777)) & 4095;
    atomicAdd(h + s, 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = h[5];
}
template <int MODE> float run(float* a, int64_t nops, uint32_t nslots, float* sink) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 8, 256>>>(a, nops, nslots, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE><<<148 * 8, 256>>>(a, nops, nslots, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
  float* a; float* sink; cudaMalloc(&a, 64 << 20); cudaMalloc(&sink, 4096 * 4);
  cudaMemset(a, 0, 64 << 20);
  const int64_t n = 40000000;
  const uint32_t slots = 1000000;  // 1M vertices
  printf("f32 RED     %.3f ms\n", run<0>(a, n, slots * 4, sink));
  printf("u32 RED     %.3f ms\n", run<5>(a, n, slots * 4, sink));
  printf("float2 RED  %.3f ms\n", run<6>(a, n, slots * 2, sink));
  printf("float4 RED  %.3f ms\n", run<1>(a, n, slots, sink));
  printf("u64 RED     %.3f ms\n", run<2>(a, n, slots * 2, sink));
  printf("f64 RED     %.3f ms\n", run<3>(a, n, slots * 2, sink));
  printf("float4 ATOM %.3f ms\n", run<4>(a, n, slots, sink));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ks<0><<<148 * 4, 512>>>(sink, n / (148 * 4));
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("smem u32 atomics (40M, 4096 bins) %.3f ms\n", ms);
  return 0;
}
