// Microbenchmark: the fast sparse-filter kernel's jump-table dispatch loop on B200,
// isolated from TMA, the ring and the epilogue.  Each warp walks 64 channels of a smem
// entry list through the generated sf3x3_chunk (8 chunks of 8 channels, patch reloaded
// per channel) with either `per` random entries per channel or Binomial(36, DENSITY).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/brx_bench tools/brx_bench.cu
//   tools/brx_bench PER [FIXED_TAP]          (FIXED_TAP >= 0: every entry the same case)
//   tools/brx_bench 0 -1 0 DENSITY
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#ifndef DISPATCH_INC
#define DISPATCH_INC "../paper_2212_08815_b200/csrc/sf3x3_dispatch.inc"
#endif
#include DISPATCH_INC
#ifndef FSCNN_SF3_KT
#define FSCNN_SF3_KT 4
#endif

template <int MASK>
__global__ void __launch_bounds__(512, 1) bench(const int2 *ents_g, int n_ent, int reps, float *out, long long *cyc, const int *starts_g) {
    __shared__ int starts[8];
    if (threadIdx.x < 8) starts[threadIdx.x] = starts_g[threadIdx.x];
    extern __shared__ int2 sm[];
    int2 *ents = sm;
    float *patch = reinterpret_cast<float *>(sm + ((n_ent + 9) & ~1));
    for (int i = threadIdx.x; i < n_ent + 8; i += blockDim.x) ents[i] = ents_g[i];
    for (int i = threadIdx.x; i < 8 * 34 * 20; i += blockDim.x) patch[i] = i * 1e-3f;
    __syncthreads();
    unsigned long long acc2[FSCNN_SF3_KT][4][2];
    for (int a = 0; a < FSCNN_SF3_KT; ++a) for (int b = 0; b < 4; ++b) acc2[a][b][0] = acc2[a][b][1] = 0;
    const int lane = threadIdx.x & 31, lx = lane & 3, ly = lane >> 2;
    uint32_t pbase = (uint32_t)__cvta_generic_to_shared(patch + (4 * ly) * 20 + 4 * lx);
    long long t0 = clock64();
    for (int rep = 0; rep < reps; ++rep) {
        uint32_t cur = (uint32_t)__cvta_generic_to_shared(ents);
        uint32_t end = cur + n_ent * 8;
        // current protocol: one call = one chunk of 8 channels, each (per) entries + sentinel slot
#pragma unroll 1
        for (int q = 0; q < 8; ++q) { sf3x3_chunk<20 * 4>(acc2, cur + 8u * starts[q], pbase, 8, 34 * 20 * 4); }
        (void)end;
    }
    long long t1 = clock64();
    float s = 0;
    for (int a = 0; a < FSCNN_SF3_KT; ++a) for (int b = 0; b < 4; ++b) for (int h = 0; h < 2; ++h) s += __uint_as_float((uint32_t)acc2[a][b][h]) + __uint_as_float((uint32_t)(acc2[a][b][h] >> 32));
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char **argv) {
    int per = argc > 1 ? atoi(argv[1]) : 4;       // nonzeros per channel
    int fixed = argc > 2 ? atoi(argv[2]) : -1;    // >= 0: every entry jumps to this case
    int n_ch = 64, reps = 50;                      // 8 chunks of 8 channels
    int n_ent = n_ch * (per + 1);
    int2 *h = (int2 *)malloc((n_ch * (FSCNN_SF3_KT * 9 + 1) + 64) * sizeof(int2));
    srand(1);
    int k = 0;
    long long binom_total = 0;
    double dens = argc > 4 ? atof(argv[4]) : 0.0;   // > 0: Binomial(KT*9, dens) distinct taps per channel
    if (dens > 0) {
        long long tot = 0;
        k = 0;
        for (int c = 0; c < n_ch; ++c) {
            int cnt = 0;
            for (int t = 0; t < FSCNN_SF3_KT * 9; ++t)
                if (rand() < dens * RAND_MAX) { h[k].x = t; float v = 1e-3f; h[k].y = *(int *)&v; ++k; ++cnt; }
            if (cnt) h[k - 1].x += FSCNN_SF3_KT * 9;
            h[k].x = cnt ? 0 : 2 * FSCNN_SF3_KT * 9; h[k].y = 0; ++k;
            tot += cnt;
        }
        n_ent = k;
        printf("binomial density %.2f: %.2f nonzeros/channel\n", dens, (double)tot / n_ch);
        per = -1; binom_total = tot;
    }
    for (int c = 0; c < n_ch && dens <= 0; ++c) {
        for (int j = 0; j < per; ++j) { h[k].x = fixed >= 0 ? fixed : rand() % (FSCNN_SF3_KT * 9); float v = 1e-3f; h[k].y = *(int *)&v; ++k; }
        if (per > 0) h[k - 1].x += FSCNN_SF3_KT * 9;   // channel-last entry falls into the transition
        h[k].x = per > 0 ? 0 : 2 * FSCNN_SF3_KT * 9; h[k].y = 0; ++k;
    }
    for (int j = 0; j < 8; ++j) { h[k + j].x = FSCNN_SF3_KT * 9; h[k + j].y = 0; }
    // chunk starts (entry index of every 8th channel)
    int hst[8];
    {
        const int NC = FSCNN_SF3_KT * 9;
        int i = 0;
        for (int c = 0; c < n_ch; ++c) {
            if (c % 8 == 0) hst[c / 8] = i;
            if (h[i].x == 2 * NC) { ++i; continue; }       // empty channel: one slot
            while (h[i].x < NC) ++i;                       // entries up to the channel-last one
            i += 2;                                        // channel-last entry + sentinel slot
        }
    }
    int *dst; cudaMalloc(&dst, 32); cudaMemcpy(dst, hst, 32, cudaMemcpyHostToDevice);
    int2 *d; float *o; long long *cyc;
    cudaMalloc(&d, (n_ent + 8) * sizeof(int2));
    cudaMemcpy(d, h, (n_ent + 8) * sizeof(int2), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    int smem = (n_ent + 10) * 8 + 8 * 34 * 20 * 4;
    auto kern = bench<0>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int warps = 4; warps <= 16; warps *= 2) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        kern<<<148, 32 * warps, smem>>>(d, n_ent, 2, o, cyc, dst);
        cudaEventRecord(a);
        kern<<<148, 32 * warps, smem>>>(d, n_ent, reps, o, cyc, dst);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        double disp = (per >= 0 ? (double)n_ch * per : (double)binom_total) * reps;
        double fl = 148.0 * warps * 32 * disp * 32;
        printf("per=%d fixed=%d warps/SM=%d: %.1f cycles/nonzero/warp, %.2f TFLOP/s (%s)\n", per, fixed, warps,
               c0 / disp, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
