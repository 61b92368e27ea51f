// Microbenchmark: shared-memory atomic throughput variants on B200.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x;
}
template <int MODE>
__global__ void ks(float* out, int64_t nops_per_block, int bins) {
  __shared__ unsigned long long h[4096];
  uint32_t* h32 = reinterpret_cast<uint32_t*>(h);
  float* hf = reinterpret_cast<float*>(h);
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) h[i] = 0;
  __syncthreads();
  uint32_t acc = 0;
  for (int64_t i = threadIdx.x; i < nops_per_block; i += blockDim.x) {
    uint32_t x = hash32((uint32_t)(i + blockIdx.x * 77777));
    uint32_t s = x & (bins - 1);
    if (MODE == 0) atomicAdd(h32 + s, x >> 20);
    if (MODE == 1) acc += atomicAdd(h32 + s, x >> 20);
    if (MODE == 2) atomicAdd(h + s, (unsigned long long)x);
    if (MODE == 3) atomicAdd(hf + s, (float)(x >> 20));
    if (MODE == 4) { acc += atomicAdd(h32 + s, 1u); }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = (float)h[5] + acc;
}
template <int MODE> void run(const char* name, float* sink, int bins) {
  const int64_t n = 40000000;
  ks<MODE><<<148 * 4, 512>>>(sink, n / (148 * 4), bins);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  ks<MODE><<<148 * 4, 512>>>(sink, n / (148 * 4), bins);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s bins %5d: %.3f ms per 40M\n", name, bins, ms);
}
int main() {
  float* sink; cudaMalloc(&sink, 1 << 20);
  for (int b : {256, 4096}) {
    run<0>("u32 add (RED)", sink, b);
    run<1>("u32 add returning", sink, b);
    run<4>("u32 inc returning", sink, b);
    run<2>("u64 add (CAS loop)", sink, b);
    run<3>("f32 add", sink, b);
  }
  return 0;
}
