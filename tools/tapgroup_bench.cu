// Microbenchmark: "tap-group" sparse-filter inner loop vs the jump-table dispatch
// (brx_bench.cu).  Per input channel a warp (4 filters x 4x4 output tile per lane)
// loads its 6x6 patch, then walks the 9 taps statically; a tap runs (all 4 filters'
// FMAs, zero weights included) only when one of the 4 filters has a nonzero there.
// No indirect branch; the cost is the FMAs on zero weights.  Timing only.
//
// usage: tapgroup_bench DENSITY   (weights ~ Bernoulli(DENSITY) per (filter, tap))
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>

__device__ __forceinline__ uint32_t warp_uniform(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

constexpr int NCH = 64, ROW = 20, CHF = 34 * ROW;  // channels, row pitch, floats per channel box

// record per channel: [mask, offset of its weight quads]; quads: float4 per active tap
__global__ void __launch_bounds__(512, 1) bench(const uint2 *rec_g, const float4 *w_g, int n_quads, int reps,
                                                float *out, long long *cyc) {
    extern __shared__ float4 sm4[];
    float4 *wq = sm4;
    uint2 *rec = reinterpret_cast<uint2 *>(wq + n_quads);
    float *patch = reinterpret_cast<float *>(rec + NCH + 2);
    for (int i = threadIdx.x; i < n_quads; i += blockDim.x) wq[i] = w_g[i];
    for (int i = threadIdx.x; i < NCH; i += blockDim.x) rec[i] = rec_g[i];
    for (int i = threadIdx.x; i < 8 * CHF; i += blockDim.x) patch[i] = i * 1e-3f;
    __syncthreads();
    float2 acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = make_float2(0.f, 0.f);
    const int lane = threadIdx.x & 31, lx = lane & 3, ly = lane >> 2;
    const float *pb = patch + (4 * ly) * ROW + 4 * lx;
    long long t0 = clock64();
#pragma unroll 1
    for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 1
        for (int ch = 0; ch < NCH; ++ch) {
            const float *pp = pb + (ch & 7) * CHF;
            float2 pt[6][3];
#pragma unroll
            for (int r = 0; r < 6; ++r) {
                const float4 a = *reinterpret_cast<const float4 *>(pp + r * ROW);
                const float2 b = *reinterpret_cast<const float2 *>(pp + r * ROW + 4);
                pt[r][0] = make_float2(a.x, a.y);
                pt[r][1] = make_float2(a.z, a.w);
                pt[r][2] = b;
            }
            const uint2 rc = rec[ch];
            const uint32_t mask = warp_uniform(rc.x);
            const float4 *wp = wq + warp_uniform(rc.y);
#pragma unroll
            for (int t = 0; t < 9; ++t) {
                if (mask & (1u << t)) {
                    const int kh = t / 3, kw = t % 3;
                    const float4 w = *wp++;
                    const float wv[4] = {w.x, w.y, w.z, w.w};
                    float2 src[4][2];
#pragma unroll
                    for (int py = 0; py < 4; ++py) {
                        if (kw == 0) { src[py][0] = pt[py + kh][0]; src[py][1] = pt[py + kh][1]; }
                        else if (kw == 2) { src[py][0] = pt[py + kh][1]; src[py][1] = pt[py + kh][2]; }
                        else {
                            src[py][0] = make_float2(pt[py + kh][0].y, pt[py + kh][1].x);
                            src[py][1] = make_float2(pt[py + kh][1].y, pt[py + kh][2].x);
                        }
                    }
#pragma unroll
                    for (int kl = 0; kl < 4; ++kl) {
                        const float2 ww = make_float2(wv[kl], wv[kl]);
#pragma unroll
                        for (int py = 0; py < 4; ++py)
#pragma unroll
                            for (int h = 0; h < 2; ++h) acc[kl][py][h] = __ffma2_rn(ww, src[py][h], acc[kl][py][h]);
                    }
                }
            }
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) s += acc[a][b][0].x + acc[a][b][0].y + acc[a][b][1].x + acc[a][b][1].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char **argv) {
    double dens = argc > 1 ? atof(argv[1]) : 0.1;
    srand(1);
    uint2 rec[NCH];
    float4 *quads = (float4 *)malloc(NCH * 9 * sizeof(float4));
    int nq = 0;
    long long nnz = 0, active = 0;
    for (int c = 0; c < NCH; ++c) {
        uint32_t mask = 0;
        rec[c].y = nq;
        for (int t = 0; t < 9; ++t) {
            float w[4];
            bool any = false;
            for (int k = 0; k < 4; ++k) {
                bool nz = rand() < dens * RAND_MAX;
                w[k] = nz ? 1e-3f : 0.f;
                nnz += nz;
                any |= nz;
            }
            if (any) { mask |= 1u << t; quads[nq++] = make_float4(w[0], w[1], w[2], w[3]); ++active; }
        }
        rec[c].x = mask;
    }
    printf("density %.2f: %.2f nonzeros/channel, %.2f active taps/channel\n", dens, (double)nnz / NCH,
           (double)active / NCH);
    uint2 *drec; float4 *dq; float *o; long long *cyc;
    cudaMalloc(&drec, sizeof(rec)); cudaMemcpy(drec, rec, sizeof(rec), cudaMemcpyHostToDevice);
    cudaMalloc(&dq, (nq + 1) * sizeof(float4)); cudaMemcpy(dq, quads, nq * sizeof(float4), cudaMemcpyHostToDevice);
    cudaMalloc(&o, 148 * 512 * 4);
    cudaMalloc(&cyc, 148 * 8);
    int smem = (nq + 1) * 16 + (NCH + 2) * 8 + 8 * CHF * 4 + 64;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int reps = 50;
    for (int warps = 4; warps <= 16; warps *= 2) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        bench<<<148, 32 * warps, smem>>>(drec, dq, nq, 2, o, cyc);
        cudaEventRecord(a);
        bench<<<148, 32 * warps, smem>>>(drec, dq, nq, reps, o, cyc);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        long long c0; cudaMemcpy(&c0, cyc, 8, cudaMemcpyDeviceToHost);
        double useful = 148.0 * warps * 32 * (double)nnz * reps * 16 * 2;  // useful FLOPs
        printf("warps/SM=%2d: %.1f cycles/channel/warp, useful %.2f TFLOP/s (%s)\n", warps,
               (double)c0 / (NCH * reps), useful / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
