// FP32 CUDA-core throughput probe: the roofline denominator for the sparse convs
// (MEASURED_PEAKS.json carries HBM and bf16 tensor peaks only).  Every thread runs
// 8 independent FFMA chains; FLOPs = 2 * 8 * 16 * iters per thread.
#include "common.cuh"

namespace fscnn {
namespace {

__global__ void __launch_bounds__(256) ffma_probe_kernel(float *out, float b, float c, int iters) {
    float a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += a[j];
    if (s == 12345.678f) out[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace
}  // namespace fscnn

extern "C" int fscnn_fp32_probe(float *out, int blocks, int iters, void *stream) {
    FSCNN_REQUIRE(out && blocks > 0 && iters > 0, "bad probe arguments");
    fscnn::ffma_probe_kernel<<<blocks, 256, 0, fscnn::as_stream(stream)>>>(out, 0.999f, 1e-4f, iters);
    FSCNN_LAUNCH_CHECK("ffma_probe_kernel");
    return FSCNN_OK;
}
