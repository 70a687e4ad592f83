// Microbenchmark: cost of the fast kernel's jump-table dispatch loop on B200,
// isolated from TMA/pipeline.  Each warp walks a smem entry list (random (kl,tap)
// entries, a sentinel every `per` entries) through sf3x3_channel_looped.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include "../paper_2212_08815_b200/csrc/sf3x3_dispatch.inc"

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(const int2 *ents_g, int n_ent, int reps, float *out, long long *cyc) {
    extern __shared__ int2 ents[];
    for (int i = threadIdx.x; i < n_ent + 4; i += blockDim.x) ents[i] = ents_g[i];
    __syncthreads();
    float acc[FSCNN_SF3_KT][4][4];
    float pt[6][6];
    for (int a = 0; a < FSCNN_SF3_KT; ++a) for (int b = 0; b < 4; ++b) for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
    for (int r = 0; r < 6; ++r) for (int c = 0; c < 6; ++c) pt[r][c] = threadIdx.x * 0.001f + r + c;
    __syncwarp();
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        uint32_t cur = (uint32_t)__cvta_generic_to_shared(ents);
        uint32_t end = cur + n_ent * 8;
        if (MODE == 0) { while (cur < end) cur = sf3x3_channel_looped(acc, pt, cur); }
        else if (MODE == 1) { while (cur < end) cur = sf3x3_channel_threaded(acc, pt, cur); }
        else if (MODE == 3) {
            const float *pbase = reinterpret_cast<const float *>(ents) + (threadIdx.x & 3) * 4 + ((threadIdx.x & 31) >> 2) * 80;
            int ch = 0;
            while (cur < end) {
                const float *rowp = pbase + (ch & 7) * 8;
#pragma unroll
                for (int r = 0; r < 6; ++r) {
                    float4 a4 = *reinterpret_cast<const float4 *>(rowp + r * 20);
                    float2 b2 = *reinterpret_cast<const float2 *>(rowp + r * 20 + 4);
                    pt[r][0] = a4.x; pt[r][1] = a4.y; pt[r][2] = a4.z; pt[r][3] = a4.w; pt[r][4] = b2.x; pt[r][5] = b2.y;
                }
                cur = sf3x3_channel_looped(acc, pt, cur);
                ++ch;
            }
        }
        else {
            // no dispatch: every entry applies case (kl = idx & 7, fixed tap) via a static
            // 8-way predicated select -- measures the loop without the indirect branch
            while (cur < end) {
                int2 e = *reinterpret_cast<int2 *>(ents + ((cur - (uint32_t)__cvta_generic_to_shared(ents)) >> 3));
                cur += 8;
                if (e.x >= FSCNN_SF3_KT * 9) continue;
                float v = __int_as_float(e.y);
#pragma unroll
                for (int py = 0; py < 4; ++py)
#pragma unroll
                    for (int px = 0; px < 4; ++px) acc[0][py][px] = fmaf(v, pt[py][px], acc[0][py][px]);
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
    for (int a = 0; a < FSCNN_SF3_KT; ++a) for (int b = 0; b < 4; ++b) for (int c = 0; c < 4; ++c) s += acc[a][b][c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char **argv) {
    int per = argc > 1 ? atoi(argv[1]) : 7;       // nonzeros per channel
    int n_ch = 64, reps = 50;
    int n_ent = n_ch * (per + 1);
    int2 *h = (int2 *)malloc((n_ent + 4) * sizeof(int2));
    srand(1);
    int k = 0;
    for (int c = 0; c < n_ch; ++c) {
        for (int j = 0; j < per; ++j) { h[k].x = rand() % (FSCNN_SF3_KT * 9); float v = 1e-3f; h[k].y = *(int *)&v; ++k; }
        h[k].x = FSCNN_SF3_KT * 9; h[k].y = 0; ++k;
    }
    for (int j = 0; j < 4; ++j) { h[k + j].x = FSCNN_SF3_KT * 9; h[k + j].y = 0; }
    int2 *d; float *o; long long *cyc;
    cudaMalloc(&d, (n_ent + 4) * sizeof(int2));
    cudaMemcpy(d, h, (n_ent + 4) * sizeof(int2), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * 32 * 16 * 4 * 8);
    cudaMalloc(&cyc, 148 * 16 * 8);
    int smem = (n_ent + 4) * 8 > 32768 ? (n_ent + 4) * 8 : 32768;
    int mode = argc > 2 ? atoi(argv[2]) : 0;
    auto kern = mode == 0 ? bench<0> : (mode == 1 ? bench<1> : (mode == 3 ? bench<3> : bench<2>));
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int warps = 4; warps <= 16; warps *= 2) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        kern<<<148, 32 * warps, smem>>>(d, n_ent, 2, o, cyc);
        cudaEventRecord(a);
        kern<<<148, 32 * warps, smem>>>(d, n_ent, reps, o, cyc);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        double disp = (double)n_ch * per * reps;  // dispatches per warp (excl. sentinels)
        double fl = 148.0 * warps * 32 * disp * 32;  // 16 FFMA x 2 FLOP per lane per dispatch
        printf("mode=%d per=%d warps/SM=%d: %.1f cycles/dispatch/warp, %.2f TFLOP/s (%s)\n", mode, per, warps,
               c0 / disp, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
