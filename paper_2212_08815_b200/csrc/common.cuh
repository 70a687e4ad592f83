// Shared helpers for the FSCNN B200 kernels: error plumbing, launch accounting,
// small device utilities.  Everything here is internal to libfscnn_b200.so.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/fscnn_b200.h"

namespace fscnn {

void set_error(const char *fmt, ...);
void note_launch(int n = 1);

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

// Check the launch that was just issued; records the error text and returns a status.
int check_launch(const char *what);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

#define FSCNN_REQUIRE(cond, ...)                        \
    do {                                                \
        if (!(cond)) {                                  \
            ::fscnn::set_error(__VA_ARGS__);            \
            return FSCNN_ERR_ARG;                       \
        }                                               \
    } while (0)

#define FSCNN_LAUNCH_CHECK(what)                        \
    do {                                                \
        int _st = ::fscnn::check_launch(what);          \
        if (_st != FSCNN_OK) return _st;                \
    } while (0)

// np.maximum(v, 0.0f): NaN propagates with its payload, -0.0 -> +0.0 (layers.py:482-483).
// Integer select so the compiler cannot turn it into FMNMX (which canonicalises NaN).
__device__ __forceinline__ float relu_np(float v) {
    const int u = __float_as_int(v);
    const bool keep = (u > 0) || ((u & 0x7fffffff) > 0x7f800000);
    return __int_as_float(keep ? u : 0);
}

// x86 float arithmetic with one NaN operand returns that operand, quieted; CUDA returns
// the canonical NaN.  Elementwise ops that must match numpy bit-for-bit (node payloads
// are compared as raw bytes) route NaNs through here.
__device__ __forceinline__ bool is_nan_bits(float v) {
    return (__float_as_int(v) & 0x7fffffff) > 0x7f800000;
}
__device__ __forceinline__ float nan_quiet(float v) { return __int_as_float(__float_as_int(v) | 0x00400000); }

}  // namespace fscnn
