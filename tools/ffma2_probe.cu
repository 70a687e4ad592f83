// FFMA vs FFMA2 (fma.rn.f32x2) throughput on B200: 8 independent chains per thread.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
__global__ void ffma(float *out, float b, float c, int iters) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
    float s = 0; for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 1.2345f) out[0] = s;
}
__global__ void ffma2(float *out, float b, float c, int iters) {
    unsigned long long a[8];
    float2 bb = make_float2(b, b), cc = make_float2(c, c);
    unsigned long long br = *reinterpret_cast<unsigned long long *>(&bb), cr = *reinterpret_cast<unsigned long long *>(&cc);
    for (int j = 0; j < 8; ++j) { float2 t = make_float2(threadIdx.x * 1e-3f + j, j); a[j] = *reinterpret_cast<unsigned long long *>(&t); }
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(br), "l"(cr));
    float s = 0; for (int j = 0; j < 8; ++j) { float2 t = *reinterpret_cast<float2 *>(&a[j]); s += t.x + t.y; }
    if (s == 1.2345f) out[0] = s;
}
int main() {
    float *o; cudaMalloc(&o, 4);
    int blocks = 148 * 8, iters = 4096;
    for (int m = 0; m < 2; ++m) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            if (m == 0) ffma<<<blocks, 256>>>(o, 0.999f, 1e-4f, iters); else ffma2<<<blocks, 256>>>(o, 0.999f, 1e-4f, iters);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double fl = (double)blocks * 256 * iters * 16 * 8 * 2 * (m ? 2 : 1);
            if (r == 2) printf("%s: %.1f TFLOP/s\n", m ? "FFMA2" : "FFMA", fl / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
