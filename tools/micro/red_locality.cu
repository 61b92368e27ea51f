// Microbenchmark: does address locality inside a warp instruction raise the
// throughput of scattered float4 RED / returning ATOM / gathers on B200?
// 40M lane operations into 1M float4 slots; groups of G consecutive lanes hit
// G consecutive slots starting at a random (G-aligned) slot.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int MODE, int G>
__global__ void k(float4* a, int64_t nops, uint32_t nslots, float* sink) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  float acc = 0.f;
  const int lane = threadIdx.x & 31;
  for (int64_t i = t; i < nops; i += stride) {
    uint32_t grp = (uint32_t)((i - lane) / 32) * (32 / G) + lane / G;
    uint32_t s = (hash32(grp) % (nslots / G)) * G + (lane % G);
    if (MODE == 0) atomicAdd(a + s, make_float4(1.f, 2.f, 3.f, 4.f));
    if (MODE == 1) { float4 o = atomicAdd(a + s, make_float4(1.f, 2.f, 3.f, 4.f)); acc += o.x; }
    if (MODE == 2) { float4 o = __ldcg(a + s); acc += o.x; }
  }
  if (acc == 12345.f) sink[0] = acc;
}
template <int MODE, int G> float run(float4* a, int64_t nops, uint32_t nslots, float* sink) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE, G><<<148 * 8, 256>>>(a, nops, nslots, sink);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<MODE, G><<<148 * 8, 256>>>(a, nops, nslots, sink);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1); return ms / 5;
}
int main() {
  float4* a; float* sink; cudaMalloc(&a, 64 << 20); cudaMalloc(&sink, 4096 * 4);
  cudaMemset(a, 0, 64 << 20);
  const int64_t n = 40000000;
  const uint32_t slots = 1 << 20;
  printf("RED  f4  G=1 %.3f  G=2 %.3f  G=4 %.3f  G=8 %.3f  G=32 %.3f ms\n", run<0, 1>(a, n, slots, sink),
         run<0, 2>(a, n, slots, sink), run<0, 4>(a, n, slots, sink), run<0, 8>(a, n, slots, sink),
         run<0, 32>(a, n, slots, sink));
  printf("ATOM f4  G=1 %.3f  G=2 %.3f  G=4 %.3f  G=8 %.3f  G=32 %.3f ms\n", run<1, 1>(a, n, slots, sink),
         run<1, 2>(a, n, slots, sink), run<1, 4>(a, n, slots, sink), run<1, 8>(a, n, slots, sink),
         run<1, 32>(a, n, slots, sink));
  printf("LDCG f4  G=1 %.3f  G=2 %.3f  G=4 %.3f  G=8 %.3f  G=32 %.3f ms\n", run<2, 1>(a, n, slots, sink),
         run<2, 2>(a, n, slots, sink), run<2, 4>(a, n, slots, sink), run<2, 8>(a, n, slots, sink),
         run<2, 32>(a, n, slots, sink));
  return 0;
}
