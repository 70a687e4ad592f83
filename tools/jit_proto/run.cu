// Runner for the straight-line sparse-filter prototype: loads k.cubin, launches the
// G group kernels concurrently (one stream each), reports nnz-TFLOP/s.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char *s; cuGetErrorString(r_, &s); printf("%s:%d %s\n", __FILE__, __LINE__, s); exit(1);} } while (0)
int main(int argc, char **argv) {
    const char *cub = argv[1];
    int G = atoi(argv[2]); long long ffma_total = atoll(argv[3]); int ctas = atoi(argv[4]); int smem = atoi(argv[5]); int nt = argc > 6 ? atoi(argv[6]) : 128; int flush = argc > 7 ? atoi(argv[7]) : 0;
    void *fl = nullptr; if (flush) cudaMalloc(&fl, (size_t)512 << 20);
    cudaFree(0);
    CUmodule m; CK(cuModuleLoad(&m, cub));
    std::vector<CUfunction> f(G);
    for (int g = 0; g < G; ++g) {
        char nm[16]; snprintf(nm, 16, "k%d", g);
        CK(cuModuleGetFunction(&f[g], m, nm));
        CK(cuFuncSetAttribute(f[g], CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, smem));
        int regs; cuFuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f[g]);
        if (g == 0) printf("regs %d\n", regs);
    }
    float *y; cudaMalloc(&y, (size_t)ctas * 512 * 4);
    std::vector<cudaStream_t> st(G);
    for (auto &s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    std::vector<cudaEvent_t> done(G); for (auto &d : done) cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
    int tiles = 0;
    for (int rep = 0; rep < 4; ++rep) {
        if (flush) cudaMemsetAsync(fl, rep, (size_t)512 << 20, 0);
        cudaEventRecord(e0, 0);
        for (int g = 0; g < G; ++g) {
            cudaStreamWaitEvent(st[g], e0, 0);
            void *args[] = {&y, &tiles};
            CK(cuLaunchKernel(f[g], ctas, 1, 1, nt, 1, 1, smem, st[g], args, nullptr));
            cudaEventRecord(done[g], st[g]);
            cudaStreamWaitEvent(0, done[g], 0);
        }
        cudaEventRecord(e1, 0); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        // each generated FFMA = 32 lanes x 2 flop per warp; ctas x 4 warps per group
        double fl = (double)ffma_total * 2.0 * 32 * (nt / 32) * ctas;
        printf("rep %d: %.3f ms  %.2f nnz-TFLOP/s  (%s)\n", rep, ms, fl / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
