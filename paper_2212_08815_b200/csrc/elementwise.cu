// Memory-bound layers between convolutions and layout converters.
//   relu      -- np.maximum(x, 0) (layers.py:469-484)
//   act       -- leaky ReLU np.where(x > 0, x, s*x) (layers.py:484) and the node-format
//                ReLU keep rule x > 0 (layers.py:488-489: NaN and -0.0 dropped)
//   batchnorm -- ((x - mean) / sqrt(var + eps)) * scale + shift (layers.py:507-509)
//   pad2d     -- zero padding of the spatial extents (layers.py:513-520)
//   pool2d    -- _pool_dense_kernel (layers.py:250-271) on NCHW
//   whc<->nchw -- DenseTensor3 memory (sparse_core.py:9-13) <-> device NCHW
//   kcrs->crsk -- dense filter bank transposed for the sparse-input kernel
// All are HBM-bound streaming kernels: grid-stride, float4 where aligned.
#include "common.cuh"

namespace fscnn {
namespace {

template <bool VEC>
__global__ void relu_kernel(const float *__restrict__ x, int64_t n, float *__restrict__ y) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t head = 0;
    if (VEC) {
        int64_t n4 = n >> 2;
        const float4 *x4 = reinterpret_cast<const float4 *>(x);
        float4 *y4 = reinterpret_cast<float4 *>(y);
        for (int64_t i = t0; i < n4; i += stride) {
            float4 v = x4[i];
            v.x = relu_np(v.x);
            v.y = relu_np(v.y);
            v.z = relu_np(v.z);
            v.w = relu_np(v.w);
            y4[i] = v;
        }
        head = n4 << 2;
    }
    for (int64_t i = head + t0; i < n; i += stride) y[i] = relu_np(x[i]);
}

// kind 1: leaky ReLU (x > 0 ? x : slope * x, one fp32 multiply like numpy);
// kind 2: the node-format ReLU keep rule, x > 0 ? x : 0 (NaN -> 0, -0.0 -> 0, so the
// re-encode drops exactly the nodes the reference drops).
__global__ void act_kernel(const float *__restrict__ x, int64_t n, int kind, float slope,
                           float *__restrict__ y) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        float v = x[i];
        if (kind == 1 && is_nan_bits(v)) y[i] = nan_quiet(v);  // numpy keeps the payload
        else y[i] = v > 0.0f ? v : (kind == 1 ? __fmul_rn(slope, v) : 0.0f);
    }
}

// NCHW, per-channel statistics; numpy's float32 op order, no contraction.
__global__ void batchnorm_kernel(const float *__restrict__ x, int64_t total, int c_n, int64_t hw,
                                 const float *__restrict__ scale, const float *__restrict__ shift,
                                 const float *__restrict__ mean, const float *__restrict__ var,
                                 float eps, float *__restrict__ y) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        int c = (int)((i / hw) % c_n);
        const float xv = x[i];
        if (is_nan_bits(xv)) {  // numpy: the NaN operand propagates, quieted
            y[i] = nan_quiet(xv);
            continue;
        }
        float sd = __fsqrt_rn(__fadd_rn(var[c], eps));
        float v = __fdiv_rn(__fsub_rn(xv, mean[c]), sd);
        y[i] = __fadd_rn(__fmul_rn(v, scale[c]), shift[c]);
    }
}

// NCHW (h, w) -> (h + 2p, w + 2p) with zeros around; one thread per output element.
__global__ void pad2d_kernel(const float *__restrict__ x, int64_t total, int h, int w, int p,
                             float *__restrict__ y) {
    const int ho = h + 2 * p, wo = w + 2 * p;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        int xo = (int)(t % wo);
        int64_t r = t / wo;
        int yo = (int)(r % ho);
        int64_t nc = r / ho;
        int xi = xo - p, yi = yo - p;
        y[t] = (xi >= 0 && xi < w && yi >= 0 && yi < h) ? x[(nc * h + yi) * (int64_t)w + xi] : 0.0f;
    }
}

// One thread per output element (n, c, ho, wo); reads the window rows (ph outer, pw inner).
__global__ void pool2d_kernel(const float *__restrict__ x, int64_t total, int h, int w, int h_p,
                              int w_p, int use_max, float *__restrict__ y) {
    int h_o = h / h_p, w_o = w / w_p;
    float area = (float)(h_p * w_p);
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        int wo = (int)(t % w_o);
        int64_t r = t / w_o;
        int ho = (int)(r % h_o);
        int64_t nc = r / h_o;
        const float *src = x + nc * h * (int64_t)w + (int64_t)(ho * h_p) * w + wo * w_p;
        float acc = use_max ? -INFINITY : 0.0f;
        for (int ph = 0; ph < h_p; ++ph)
            for (int pw = 0; pw < w_p; ++pw) {
                float v = src[(int64_t)ph * w + pw];
                if (use_max) {
                    if (v > acc) acc = v;
                } else if (!is_nan_bits(acc)) {  // numpy: the first NaN summed wins
                    acc = is_nan_bits(v) ? nan_quiet(v) : __fadd_rn(acc, v);
                }
            }
        y[t] = use_max ? acc : (is_nan_bits(acc) ? acc : __fdiv_rn(acc, area));
    }
}

// Specialised 2x2 max-pool (every VGG16 pool): float2 row reads, same -inf / '>' rule.
__global__ void maxpool2x2_kernel(const float *__restrict__ x, int64_t total, int h, int w,
                                  float *__restrict__ y) {
    int h_o = h >> 1, w_o = w >> 1;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        int wo = (int)(t % w_o);
        int64_t r = t / w_o;
        int ho = (int)(r % h_o);
        int64_t nc = r / h_o;
        const float *src = x + nc * h * (int64_t)w + (int64_t)(2 * ho) * w + 2 * wo;
        float2 a = *reinterpret_cast<const float2 *>(src);
        float2 b = *reinterpret_cast<const float2 *>(src + w);
        float acc = -INFINITY;
        if (a.x > acc) acc = a.x;
        if (a.y > acc) acc = a.y;
        if (b.x > acc) acc = b.x;
        if (b.y > acc) acc = b.y;
        y[t] = acc;
    }
}

// (W,H,C)-memory image -> NCHW, 32x32 smem transpose over (c, hw) per image.  The NCHW
// side has row pitch ld and starts at column col0 (ld = w, col0 = 0: dense; the halo
// layout of the fast kernel: ld = halo pitch, col0 = 1).
// (W,H,C) <-> NCHW: a CTA moves a tile of 32 channels x kTH rows x 32 columns.  Both
// sides are read/written 128 B at a time, and the tile's kTH pixels of one column are
// contiguous in (W,H,C) memory (so are its kTH rows of one channel in NCHW), which
// keeps each CTA's DRAM traffic inside a few pages.  (A 32-pixel x 32-channel tile along
// q = h*W + w spread its 32 (W,H,C) pixels H*C floats apart: 1.56 TB/s.)
constexpr int kTH = 4, kTPitch = 32 * kTH + 1;

__global__ void __launch_bounds__(256) whc_to_nchw_kernel(const float *__restrict__ x, int c_n, int h, int w,
                                                          int ld, int col0, float *__restrict__ y) {
    __shared__ float tile[32 * kTPitch];
    // channel tiles of one pixel tile are launched back to back (they share DRAM pages
    // on the (W,H,C) side)
    const int n_ct = (c_n + 31) / 32, n_wt = (w + 31) / 32;
    const int c0 = (blockIdx.x % n_ct) * 32, pt = blockIdx.x / n_ct;
    const int w0 = (pt % n_wt) * 32, h0 = (pt / n_wt) * kTH;
    const int img = blockIdx.z, tx = threadIdx.x;
    const float *src = x + (int64_t)img * c_n * h * w;
    float *dst = y + (int64_t)img * c_n * h * ld + col0;
#pragma unroll
    for (int r = threadIdx.y; r < 32 * kTH; r += 8) {  // r = (w_l, h_l): loads along c
        const int wl = r / kTH, hl = r % kTH;
        if (w0 + wl < w && h0 + hl < h && c0 + tx < c_n)
            tile[tx * kTPitch + hl * 32 + wl] = src[((int64_t)(w0 + wl) * h + h0 + hl) * c_n + c0 + tx];
    }
    __syncthreads();
#pragma unroll
    for (int r = threadIdx.y; r < 32 * kTH; r += 8) {  // r = (c_l, h_l): stores along w
        const int cl = r / kTH, hl = r % kTH;
        if (w0 + tx < w && h0 + hl < h && c0 + cl < c_n)
            dst[((int64_t)(c0 + cl) * h + h0 + hl) * ld + w0 + tx] = tile[cl * kTPitch + hl * 32 + tx];
    }
}

// Shallow images: one thread per output pixel (img, h, w) in NCHW order, so the c
// plane writes coalesce; the (W,H,C) reads are C-float strided.
__global__ void whc_to_nchw_small_kernel(const float *__restrict__ x, int64_t total, int c_n, int h, int w,
                                         int ld, int col0, float *__restrict__ y) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int wi = (int)(t % w);
        const int64_t r = t / w;
        const int hi = (int)(r % h);
        const int64_t img = r / h;
        const float *src = x + ((img * w + wi) * (int64_t)h + hi) * c_n;
        float *dst = y + (img * c_n * h + hi) * (int64_t)ld + col0 + wi;
        for (int c = 0; c < c_n; ++c) dst[(int64_t)c * h * ld] = src[c];
    }
}

__global__ void __launch_bounds__(256) nchw_to_whc_kernel(const float *__restrict__ x, int c_n, int h, int w,
                                                          int ld, int col0, float *__restrict__ y) {
    __shared__ float tile[32 * kTPitch];
    // channel tiles of one pixel tile are launched back to back (they share DRAM pages
    // on the (W,H,C) side)
    const int n_ct = (c_n + 31) / 32, n_wt = (w + 31) / 32;
    const int c0 = (blockIdx.x % n_ct) * 32, pt = blockIdx.x / n_ct;
    const int w0 = (pt % n_wt) * 32, h0 = (pt / n_wt) * kTH;
    const int img = blockIdx.z, tx = threadIdx.x;
    const float *src = x + (int64_t)img * c_n * h * ld + col0;
    float *dst = y + (int64_t)img * c_n * h * w;
#pragma unroll
    for (int r = threadIdx.y; r < 32 * kTH; r += 8) {  // r = (c_l, h_l): loads along w
        const int cl = r / kTH, hl = r % kTH;
        if (w0 + tx < w && h0 + hl < h && c0 + cl < c_n)
            tile[cl * kTPitch + hl * 32 + tx] = src[((int64_t)(c0 + cl) * h + h0 + hl) * ld + w0 + tx];
    }
    __syncthreads();
#pragma unroll
    for (int r = threadIdx.y; r < 32 * kTH; r += 8) {  // r = (w_l, h_l): stores along c
        const int wl = r / kTH, hl = r % kTH;
        if (w0 + wl < w && h0 + hl < h && c0 + tx < c_n)
            dst[((int64_t)(w0 + wl) * h + h0 + hl) * c_n + c0 + tx] = tile[tx * kTPitch + hl * 32 + wl];
    }
}

// Narrow images (W < 32): 32 channels x 32 pixels taken along q = h*W + w.
__global__ void whc_to_nchw_q_kernel(const float *__restrict__ x, int c_n, int hw, int h, int w,
                                   int ld, int col0, float *__restrict__ y) {
    // tile = 32 channels x 32 pixels, pixels enumerated in the destination's (h, w)
    // order: the loads run along c (contiguous in (W,H,C)), the stores along w
    __shared__ float tile[32][33];
    int img = blockIdx.z;
    const float *src = x + (int64_t)img * c_n * hw;
    float *dst = y + (int64_t)img * c_n * h * ld + col0;
    int c0 = blockIdx.y * 32, q0 = blockIdx.x * 32;  // q = h*W + w
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int q = q0 + j, c = c0 + threadIdx.x;
        if (q < hw && c < c_n) {
            int hi = q / w, wi = q - hi * w;
            tile[j][threadIdx.x] = src[((int64_t)wi * h + hi) * c_n + c];
        }
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int c = c0 + j, q = q0 + threadIdx.x;
        if (q < hw && c < c_n) {
            int hi = q / w, wi = q - hi * w;
            dst[((int64_t)c * h + hi) * ld + wi] = tile[threadIdx.x][j];
        }
    }
}


__global__ void nchw_to_whc_q_kernel(const float *__restrict__ x, int c_n, int hw, int h, int w,
                                   int ld, int col0, float *__restrict__ y) {
    __shared__ float tile[32][33];
    int img = blockIdx.z;
    const float *src = x + (int64_t)img * c_n * h * ld + col0;
    float *dst = y + (int64_t)img * c_n * hw;
    int c0 = blockIdx.y * 32, q0 = blockIdx.x * 32;  // q = h*W + w in source order
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int c = c0 + j, q = q0 + threadIdx.x;
        if (q < hw && c < c_n) tile[j][threadIdx.x] = src[((int64_t)c * h + q / w) * ld + q % w];
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        int q = q0 + j, c = c0 + threadIdx.x;
        if (q < hw && c < c_n) {
            int hi = q / w, wi = q % w;
            dst[((int64_t)wi * h + hi) * c_n + c] = tile[threadIdx.x][j];
        }
    }
}

__global__ void kcrs_to_crsk_kernel(const float *__restrict__ src, int k_n, int crs,
                                    float *__restrict__ dst) {
    int64_t total = (int64_t)k_n * crs;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        int k = (int)(t % k_n);
        int64_t j = t / k_n;
        dst[t] = src[(int64_t)k * crs + j];
    }
}

inline unsigned grid_for(int64_t n, int threads) {
    int64_t b = ceil_div(n, threads);
    return (unsigned)(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}

// Row-pitched copy: rows of w floats from x (pitch ldx, first column colx) to y (pitch
// ldy, first column coly) -- dense NCHW <-> the halo-column activation layout.  One warp
// per row segment of 32 floats.
__global__ void pitch_copy_kernel(const float *__restrict__ x, int64_t rows, int w, int ldx, int colx,
                                  float *__restrict__ y, int ldy, int coly) {
    const int segs = (w + 31) >> 5;
    const int64_t total = rows * segs;
    const int64_t stride = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (int64_t t = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); t < total; t += stride) {
        const int64_t r = t / segs;
        const int col = (int)(t % segs) * 32 + lane;
        if (col < w) y[r * ldy + coly + col] = x[r * ldx + colx + col];
    }
}

}  // namespace
}  // namespace fscnn

using namespace fscnn;

extern "C" {

int fscnn_relu(const float *x, int64_t count, float *y, void *stream) {
    FSCNN_REQUIRE(count >= 0 && (count == 0 || (x && y)), "bad relu arguments");
    if (count == 0) return FSCNN_OK;
    bool aligned = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
    if (aligned)
        relu_kernel<true><<<grid_for(count / 4 + 1, 256), 256, 0, as_stream(stream)>>>(x, count, y);
    else
        relu_kernel<false><<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(x, count, y);
    FSCNN_LAUNCH_CHECK("relu_kernel");
    return FSCNN_OK;
}

int fscnn_activation(const float *x, int64_t count, int kind, float slope, float *y,
                     void *stream) {
    FSCNN_REQUIRE(count >= 0 && (count == 0 || (x && y)), "bad activation arguments");
    FSCNN_REQUIRE(kind >= 0 && kind <= 2, "unknown activation kind");
    if (kind == 0) return fscnn_relu(x, count, y, stream);
    if (count == 0) return FSCNN_OK;
    act_kernel<<<grid_for(count, 256), 256, 0, as_stream(stream)>>>(x, count, kind, slope, y);
    FSCNN_LAUNCH_CHECK("act_kernel");
    return FSCNN_OK;
}

int fscnn_batchnorm(const float *x, int n, int c, int h, int w, const float *scale,
                    const float *shift, const float *mean, const float *var, float eps, float *y,
                    void *stream) {
    FSCNN_REQUIRE(n >= 0 && c >= 0 && h >= 0 && w >= 0, "negative extent");
    int64_t total = (int64_t)n * c * h * w;
    if (total == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && y && scale && shift && mean && var, "null buffer");
    batchnorm_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(
        x, total, c, (int64_t)h * w, scale, shift, mean, var, eps, y);
    FSCNN_LAUNCH_CHECK("batchnorm_kernel");
    return FSCNN_OK;
}

int fscnn_pad2d(const float *x, int n, int c, int h, int w, int p, float *y, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c >= 0 && h >= 0 && w >= 0, "negative extent");
    FSCNN_REQUIRE(p >= 0, "pad width must be non-negative");
    int64_t total = (int64_t)n * c * (h + 2 * p) * (w + 2 * p);
    if (total == 0) return FSCNN_OK;
    FSCNN_REQUIRE(y && (x || (int64_t)n * c * h * w == 0), "null buffer");
    pad2d_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(x, total, h, w, p, y);
    FSCNN_LAUNCH_CHECK("pad2d_kernel");
    return FSCNN_OK;
}

int fscnn_pool2d(const float *x, int n, int c, int h, int w, int h_p, int w_p, int use_max,
                 float *y, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c >= 0 && h >= 0 && w >= 0, "negative extent");
    FSCNN_REQUIRE(h_p > 0 && w_p > 0, "pool window must be positive");
    FSCNN_REQUIRE(h % h_p == 0 && w % w_p == 0, "input not divisible by pool window");
    int64_t total = (int64_t)n * c * (h / h_p) * (w / w_p);
    if (total == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && y, "null buffer");
    bool even_rows = (w % 2 == 0) && ((reinterpret_cast<uintptr_t>(x) & 7) == 0);
    if (use_max && h_p == 2 && w_p == 2 && even_rows) {
        maxpool2x2_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(x, total, h, w, y);
        FSCNN_LAUNCH_CHECK("maxpool2x2_kernel");
    } else {
        pool2d_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(x, total, h, w, h_p, w_p,
                                                                          use_max, y);
        FSCNN_LAUNCH_CHECK("pool2d_kernel");
    }
    return FSCNN_OK;
}

int fscnn_whc_to_nchw_ex(const float *x_whc, int n, int c, int h, int w, float *y, int ld,
                         int col0, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c >= 0 && h >= 0 && w >= 0, "negative extent");
    FSCNN_REQUIRE(col0 >= 0 && ld >= w + col0, "row pitch too small");
    if ((int64_t)n * c * h * w == 0) return FSCNN_OK;
    if (c <= 8) {  // shallow images (the network input): a thread per pixel, no smem tile
        const int64_t total = (int64_t)n * h * w;
        whc_to_nchw_small_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(x_whc, total, c, h, w,
                                                                                      ld, col0, y);
        FSCNN_LAUNCH_CHECK("whc_to_nchw_small_kernel");
        return FSCNN_OK;
    }
    if (w < 32) {
        dim3 grid((unsigned)ceil_div((int64_t)h * w, 32), (unsigned)ceil_div(c, 32), (unsigned)n);
        whc_to_nchw_q_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(x_whc, c, h * w, h, w, ld, col0, y);
        FSCNN_LAUNCH_CHECK("whc_to_nchw_q_kernel");
        return FSCNN_OK;
    }
    dim3 grid((unsigned)(ceil_div(w, 32) * ceil_div(h, kTH) * ceil_div(c, 32)), 1, (unsigned)n);
    whc_to_nchw_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(x_whc, c, h, w, ld, col0, y);
    FSCNN_LAUNCH_CHECK("whc_to_nchw_kernel");
    return FSCNN_OK;
}

int fscnn_whc_to_nchw(const float *x_whc, int n, int c, int h, int w, float *y_nchw,
                      void *stream) {
    return fscnn_whc_to_nchw_ex(x_whc, n, c, h, w, y_nchw, w, 0, stream);
}

int fscnn_nchw_to_whc_ex(const float *x, int n, int c, int h, int w, int ld, int col0, float *y_whc,
                         void *stream) {
    FSCNN_REQUIRE(n >= 0 && c >= 0 && h >= 0 && w >= 0, "negative extent");
    FSCNN_REQUIRE(col0 >= 0 && ld >= w + col0, "row pitch too small");
    if ((int64_t)n * c * h * w == 0) return FSCNN_OK;
    if (w < 32) {
        dim3 grid((unsigned)ceil_div((int64_t)h * w, 32), (unsigned)ceil_div(c, 32), (unsigned)n);
        nchw_to_whc_q_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(x, c, h * w, h, w, ld, col0, y_whc);
        FSCNN_LAUNCH_CHECK("nchw_to_whc_q_kernel");
        return FSCNN_OK;
    }
    dim3 grid((unsigned)(ceil_div(w, 32) * ceil_div(h, kTH) * ceil_div(c, 32)), 1, (unsigned)n);
    nchw_to_whc_kernel<<<grid, dim3(32, 8), 0, as_stream(stream)>>>(x, c, h, w, ld, col0, y_whc);
    FSCNN_LAUNCH_CHECK("nchw_to_whc_kernel");
    return FSCNN_OK;
}

int fscnn_nchw_to_whc(const float *x_nchw, int n, int c, int h, int w, float *y_whc,
                      void *stream) {
    return fscnn_nchw_to_whc_ex(x_nchw, n, c, h, w, w, 0, y_whc, stream);
}

int fscnn_kcrs_to_crsk(const float *w_kcrs, int k, int c, int r, int s, float *w_crsk,
                       void *stream) {
    FSCNN_REQUIRE(k > 0 && c > 0 && r > 0 && s > 0 && w_kcrs && w_crsk, "bad transpose arguments");
    int64_t total = (int64_t)k * c * r * s;
    kcrs_to_crsk_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(w_kcrs, k, c * r * s,
                                                                            w_crsk);
    FSCNN_LAUNCH_CHECK("kcrs_to_crsk_kernel");
    return FSCNN_OK;
}

int fscnn_pitch_copy(const float *x, int64_t rows, int w, int ldx, int colx, float *y, int ldy,
                     int coly, void *stream) {
    FSCNN_REQUIRE(rows >= 0 && w >= 0 && colx >= 0 && coly >= 0, "negative extent");
    FSCNN_REQUIRE(ldx >= w + colx && ldy >= w + coly, "row pitch too small");
    if (rows == 0 || w == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && y, "null buffer");
    const int64_t warps = rows * ((w + 31) / 32);
    const int64_t blocks = (warps + 7) / 8;
    pitch_copy_kernel<<<(unsigned)(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, as_stream(stream)>>>(
        x, rows, w, ldx, colx, y, ldy, coly);
    FSCNN_LAUNCH_CHECK("pitch_copy_kernel");
    return FSCNN_OK;
}

}  // extern "C"
