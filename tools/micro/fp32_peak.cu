// FP32 CUDA-core peak on this B200: scalar FFMA and packed FFMA2 (fma.rn.f32x2)
// throughput, 8 independent chains per thread, 148 x 8 CTAs of 256 threads.
// Flops counted as 2 per FMA lane-op (FFMA2: 4 per instruction per lane).
#include <cstdio>
#include <cuda_runtime.h>

template <bool PACKED>
__global__ void __launch_bounds__(256) k(float* out, int iters, float a) {
    float x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
        if (PACKED) {
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
                unsigned long long v, m;
                asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(x[i]), "f"(x[i + 1]));
                asm("mov.b64 %0, {%1, %1};" : "=l"(m) : "f"(a));
                asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v) : "l"(m));
                asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v) : "l"(m));
                asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v) : "l"(m));
                asm("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v) : "l"(m));
                asm("mov.b64 {%0, %1}, %2;" : "=f"(x[i]), "=f"(x[i + 1]) : "l"(v));
            }
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                x[i] = fmaf(x[i], a, a);
                x[i] = fmaf(x[i], a, a);
                x[i] = fmaf(x[i], a, a);
                x[i] = fmaf(x[i], a, a);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1234.5f) out[0] = s;
}

int main() {
    float* out;
    cudaMalloc(&out, 4);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int packed = 0; packed < 2; ++packed) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(e0);
            if (packed) k<true><<<blocks, threads>>>(out, iters, 0.999f);
            else k<false><<<blocks, threads>>>(out, iters, 0.999f);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            // 16 values x 4 FMA per iteration per thread, 2 flops each
            const double flops = 2.0 * 16 * 4 * (double)iters * blocks * threads;
            if (rep == 2) printf("%s: %.1f TFLOP/s (%.3f ms)\n", packed ? "FFMA2 (fma.rn.f32x2)" : "FFMA", flops / ms / 1e9, ms);
        }
    }
    return 0;
}
