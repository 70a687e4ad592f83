// Minimal TMA sanity test: 4D fp32 box load into shared memory, compare to host.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__global__ void k(const __grid_constant__ CUtensorMap tmap, float *out, int nfl, int x0, int y0) {
    extern __shared__ __align__(1024) unsigned char sm[];
    float *buf = reinterpret_cast<float *>(sm);
    __shared__ __align__(8) unsigned long long bar;
    uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nfl * 4) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"((uint32_t)__cvta_generic_to_shared(buf)),
            "l"(reinterpret_cast<uint64_t>(&tmap)), "r"(x0), "r"(y0), "r"(0), "r"(0), "r"(b)
            : "memory");
    }
    asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@!P1 bra W;\n}\n" ::"r"(b) : "memory");
    for (int i = threadIdx.x; i < nfl; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char **argv) {
    int W = 56, H = 56, C = 64, N = 1, BW = 20, BH = 10, BC = 8;
    int x0 = argc > 1 ? atoi(argv[1]) : -1, y0 = argc > 2 ? atoi(argv[2]) : -1;
    std::vector<float> h((size_t)N * C * H * W);
    for (size_t i = 0; i < h.size(); ++i) h[i] = (float)i;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    int nfl = BW * BH * BC;
    cudaMalloc(&o, nfl * 4);
    void *fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    printf("entry point: %d %d %p\n", (int)e, (int)q, fp);
    CUtensorMap map;
    cuuint64_t gdim[4] = {(cuuint64_t)W, (cuuint64_t)H, (cuuint64_t)C, (cuuint64_t)N};
    cuuint64_t gstr[3] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4, (cuuint64_t)W * H * C * 4};
    cuuint32_t box[4] = {(cuuint32_t)BW, (cuuint32_t)BH, (cuuint32_t)BC, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = ((EncodeTiledFn)fp)(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, d, gdim, gstr, box, es,
                                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    k<<<1, 128, 64 * 1024>>>(map, o, nfl, x0, y0);
    e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> got(nfl);
    cudaMemcpy(got.data(), o, nfl * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int c = 0; c < BC; ++c)
        for (int y = 0; y < BH; ++y)
            for (int x = 0; x < BW; ++x) {
                int gx = x0 + x, gy = y0 + y;
                float want = (gx >= 0 && gx < W && gy >= 0 && gy < H) ? h[((size_t)c * H + gy) * W + gx] : 0.f;
                if (got[(c * BH + y) * BW + x] != want) ++bad;
            }
    printf("mismatches: %d of %d\n", bad, nfl);
    return 0;
}
