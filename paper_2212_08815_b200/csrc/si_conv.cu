// Sparse-Input convolution, bit-exact with _conv_input_sparse_kernel
// (kernels.py:136-166) for all K filters of a layer at once.
//
// Gather form over the reference's CHW node format: output (n, k, i, j) walks
// taps kw outer, kh inner, and the input channel fiber at (w_in, h_in) in ascending
// c, accumulating filt[k][c][kh][kw] * v with separate fp32 multiply and add.
// Mapping: a warp owns one output pixel and 32 consecutive filters (lane = k), so
// the node stream is warp-uniform (broadcast loads) and the weight loads from the
// transposed [c][kh][kw][K] bank are one coalesced 128-byte line per node.
// Results equal to zero are written as +0.0 (the reference stores no node and
// densify yields +0.0), then + bias[k] when a bias is given (layers.py:425-428).
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"

namespace fscnn {
namespace {

constexpr int kPixPerBlock = 8;  // warps per block, one output pixel each

// Calls f(c, v) for the nodes of segment s in order (the reference's fiber walk).  The
// segments are consecutive (seg_off[s + 1] = seg_off[s] + count + 1, the sentinel last),
// so the fiber's length is known up front: the warp reads it 32 nodes per coalesced load
// and broadcasts them, instead of a chain of dependent single-node loads (one L2 round
// trip per node, the latency that bounds a one-image layer).  COOP = false keeps the
// single-node walk: with a full GPU of warps the latency is hidden and the two shuffles
// per node cost more (batch 32: 1.5-2x slower with COOP, measured).  The batch's last segment
// has no successor offset and keeps the sentinel walk.  Warp-uniform: every lane calls f
// for every node.
template <bool COOP, typename F>
__device__ __forceinline__ void walk_fiber(const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off,
                                           int64_t s, int64_t n_seg, int lane, F &&f) {
    int64_t q = seg_off[s];
    if (COOP && s + 1 < n_seg) {
        const int64_t e = seg_off[s + 1] - 1;
        for (; q < e; q += 32) {
            const int cnt = (int)(e - q < 32 ? e - q : 32);
            int2 mine = make_int2(0, 0);
            if (lane < cnt) mine = nodes[q + lane];
            for (int t = 0; t < cnt; ++t)
                f(__shfl_sync(0xffffffffu, mine.x, t), __int_as_float(__shfl_sync(0xffffffffu, mine.y, t)));
        }
    } else {
        for (int2 nd = nodes[q]; nd.x != -1; nd = nodes[++q]) f(nd.x, __int_as_float(nd.y));
    }
}

__global__ void __launch_bounds__(kPixPerBlock * 32)
    si_gather_kernel(const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off, int c_n,
                     int h_i, int w_i, const float *__restrict__ wt, int k_n, int h_f, int w_f,
                     int stride, int pad, int n_h, int n_w, const float *__restrict__ bias,
                     float *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int pix = blockIdx.x * kPixPerBlock + (threadIdx.x >> 5);
    const int k = blockIdx.y * 32 + lane;
    const int img = blockIdx.z;
    if (pix >= n_h * n_w) return;
    const int i = pix / n_w, j = pix % n_w;
    const int64_t *so = seg_off + (int64_t)img * h_i * w_i;
    const bool live = k < k_n;
    float acc = 0.0f;
    for (int l = 0; l < w_f; ++l) {
        int w_in = l + j * stride - pad;
        if (w_in < 0 || w_in >= w_i) continue;
        for (int kk = 0; kk < h_f; ++kk) {
            int h_in = kk + i * stride - pad;
            if (h_in < 0 || h_in >= h_i) continue;
            int64_t q = so[(int64_t)w_in * h_i + h_in];
            const float *wrow = wt + ((int64_t)kk * w_f + l) * k_n + (live ? k : 0);
            const int64_t cstride = (int64_t)h_f * w_f * k_n;
            for (int2 nd = nodes[q]; nd.x != -1; nd = nodes[++q]) {
                float wv = wrow[(int64_t)nd.x * cstride];
                acc = __fadd_rn(acc, __fmul_rn(wv, __int_as_float(nd.y)));
            }
        }
    }
    if (!live) return;
    float v = (acc != 0.0f) ? acc : 0.0f;
    if (bias) v = __fadd_rn(v, bias[k]);
    y[(((int64_t)img * k_n + k) * n_h + i) * n_w + j] = v;
}

// 3x3 / stride 1 / pad 1 strip kernel (every VGG16 shape).  A warp owns 32 filters
// (lane = k) and a strip of S consecutive outputs (i, j0..j0+S-1).  It walks the
// strip's input columns w_in = j0-1 .. j0+S left to right and, within a column, rows
// h_in = i-1 .. i+1, then the column's channel fiber.  For output j' the tap of
// column w_in is l = w_in - j' + 1, so each output sees its contributions with l
// ascending (outer), kh ascending, c ascending -- the reference order -- and the
// sums are bit-identical.  Each node loads its three kw weights for this lane with
// one 16-byte load from the [c][kh][K][4] bank and updates up to three outputs.
template <int S>
__global__ void __launch_bounds__(128, 8)
    si_strip_kernel(const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off, int c_n,
                    int h_i, int w_i, const float4 *__restrict__ wq, int k_n, int strips,
                    const float *__restrict__ bias, float *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int job = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (job >= h_i * strips) return;
    const int i = job / strips, j0 = (job % strips) * S;
    const int k = blockIdx.y * 32 + lane;
    const int img = blockIdx.z;
    const bool live = k < k_n;
    const int kq = live ? k : 0;
    const int64_t seg0 = (int64_t)img * h_i * w_i, n_seg = (int64_t)gridDim.z * h_i * w_i;
    float acc[S];
#pragma unroll
    for (int t = 0; t < S; ++t) acc[t] = 0.0f;
#pragma unroll
    for (int col = 0; col < S + 2; ++col) {
        const int w_in = j0 - 1 + col;
        if (w_in < 0 || w_in >= w_i) continue;
#pragma unroll
        for (int kk = 0; kk < 3; ++kk) {
            const int h_in = i - 1 + kk;
            if (h_in < 0 || h_in >= h_i) continue;
            walk_fiber<false>(nodes, seg_off, seg0 + (int64_t)w_in * h_i + h_in, n_seg, lane, [&](int ch, float v) {
                const float4 wv = wq[((int64_t)ch * 3 + kk) * k_n + kq];
                // output j' = col - l (strip-relative), tap l = 0,1,2
#pragma unroll
                for (int l = 0; l < 3; ++l) {
                    const int jp = col - l;
                    if (jp < 0 || jp >= S) continue;
                    const float w = l == 0 ? wv.x : (l == 1 ? wv.y : wv.z);
                    acc[jp] = __fadd_rn(acc[jp], __fmul_rn(w, v));
                }
            });
        }
    }
    if (!live) return;
#pragma unroll
    for (int t = 0; t < S; ++t) {
        const int j = j0 + t;
        if (j >= w_i) break;
        float v = (acc[t] != 0.0f) ? acc[t] : 0.0f;
        if (bias) v = __fadd_rn(v, bias[k]);
        y[(((int64_t)img * k_n + k) * h_i + i) * w_i + j] = v;
    }
}

// Shallow-bank variant (C <= 128): the strip kernel's weight loads dominate it (L2-bound,
// 16 B per node per lane).  Here a persistent CTA keeps its 32-filter block's whole
// [c][kh][32] float4 bank in shared memory (1.5 KB per channel) and walks many strips, so
// every weight comes from shared memory; per-output order and arithmetic are the strip
// kernel's (bit-exact).
template <int S, bool COOP>
__global__ void __launch_bounds__(512)
    si_strip_smem_kernel(const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off, int n_img,
                         int c_n, int h_i, int w_i, const float4 *__restrict__ wq, int k_n, int strips,
                         const float *__restrict__ bias, float *__restrict__ y) {
    extern __shared__ float4 ws[];  // [c_n * 3][32]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const int k = blockIdx.y * 32 + lane;
    const bool live = k < k_n;
    // stage the bank with cp.async (all of a thread's 16-byte copies in flight at once;
    // filters past K zero-filled)
    const uint32_t ws0 = (uint32_t)__cvta_generic_to_shared(ws);
    for (int idx = threadIdx.x; idx < c_n * 3 * 32; idx += blockDim.x) {
        const int row = idx >> 5, kk = blockIdx.y * 32 + (idx & 31);
        const float4 *src = wq + (int64_t)row * k_n + (kk < k_n ? kk : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ws0 + idx * 16), "l"(src),
                     "r"(kk < k_n ? 16 : 0)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    const int64_t jobs = (int64_t)n_img * h_i * strips;
    // one-image problems deal jobs round-robin over the CTAs (job = warp * grid + cta): a
    // grid sized to the SMs then keeps every SM busy with fewer jobs than warps (config 2:
    // 15 -> 13 us); large ones keep consecutive jobs (shared input rows) in a CTA
    const int64_t j_first = COOP ? (int64_t)warp * gridDim.x + blockIdx.x : (int64_t)blockIdx.x * nwarp + warp;
    for (int64_t job = j_first; job < jobs; job += (int64_t)gridDim.x * nwarp) {
        const int img = (int)(job / ((int64_t)h_i * strips));
        const int rem = (int)(job % ((int64_t)h_i * strips));
        const int i = rem / strips, j0 = (rem % strips) * S;
        const int64_t seg0 = (int64_t)img * h_i * w_i, n_seg = (int64_t)n_img * h_i * w_i;
        float acc[S];
#pragma unroll
        for (int t = 0; t < S; ++t) acc[t] = 0.0f;
        if constexpr (COOP && S <= 4) {
            // one-image problems: issue every fiber's offsets, then every fiber's first 32
            // nodes, before any arithmetic (two L2 round trips per job instead of two per
            // fiber); then the reference-order walk over the registers
            constexpr int NF = (S + 2) * 3;
            int64_t fq[NF], fe[NF];
            int2 fm[NF];
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int w_in = j0 - 1 + f / 3, h_in = i - 1 + f % 3;
                const bool ok = w_in >= 0 && w_in < w_i && h_in >= 0 && h_in < h_i;
                const int64_t sg = seg0 + (int64_t)w_in * h_i + h_in;
                fq[f] = ok ? seg_off[sg] : 0;
                fe[f] = !ok ? 0 : (sg + 1 < n_seg ? seg_off[sg + 1] - 1 : -1);  // -1: walk to the sentinel
            }
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int64_t cnt = fe[f] < 0 ? 0 : fe[f] - fq[f];
                fm[f] = lane < cnt ? nodes[fq[f] + lane] : make_int2(0, 0);
            }
#pragma unroll
            for (int f = 0; f < NF; ++f) {
                const int col = f / 3, kk = f % 3;
                auto apply = [&](int ch, float v) {
                    const float4 wv = ws[(ch * 3 + kk) * 32 + lane];
#pragma unroll
                    for (int l = 0; l < 3; ++l) {
                        const int jp = col - l;
                        if (jp < 0 || jp >= S) continue;
                        const float wl = l == 0 ? wv.x : (l == 1 ? wv.y : wv.z);
                        acc[jp] = __fadd_rn(acc[jp], __fmul_rn(wl, v));
                    }
                };
                if (fe[f] < 0) {
                    int64_t q = fq[f];
                    for (int2 nd = nodes[q]; nd.x != -1; nd = nodes[++q]) apply(nd.x, __int_as_float(nd.y));
                    continue;
                }
                int2 mine = fm[f];
                for (int64_t q = fq[f]; q < fe[f]; q += 32) {
                    const int cnt = (int)(fe[f] - q < 32 ? fe[f] - q : 32);
                    if (q != fq[f]) mine = lane < cnt ? nodes[q + lane] : make_int2(0, 0);
#pragma unroll 4
                    for (int t = 0; t < cnt; ++t)
                        apply(__shfl_sync(0xffffffffu, mine.x, t), __int_as_float(__shfl_sync(0xffffffffu, mine.y, t)));
                }
            }
        } else {
#pragma unroll
        for (int col = 0; col < S + 2; ++col) {
            const int w_in = j0 - 1 + col;
            if (w_in < 0 || w_in >= w_i) continue;
#pragma unroll
            for (int kk = 0; kk < 3; ++kk) {
                const int h_in = i - 1 + kk;
                if (h_in < 0 || h_in >= h_i) continue;
                walk_fiber<COOP>(nodes, seg_off, seg0 + (int64_t)w_in * h_i + h_in, n_seg, lane, [&](int ch, float v) {
                    const float4 wv = ws[(ch * 3 + kk) * 32 + lane];
#pragma unroll
                    for (int l = 0; l < 3; ++l) {
                        const int jp = col - l;
                        if (jp < 0 || jp >= S) continue;
                        const float wl = l == 0 ? wv.x : (l == 1 ? wv.y : wv.z);
                        acc[jp] = __fadd_rn(acc[jp], __fmul_rn(wl, v));
                    }
                });
            }
        }
        }
        if (!live) continue;
#pragma unroll
        for (int t = 0; t < S; ++t) {
            const int j = j0 + t;
            if (j >= w_i) break;
            float v = (acc[t] != 0.0f) ? acc[t] : 0.0f;
            if (bias) v = __fadd_rn(v, bias[k]);
            y[(((int64_t)img * k_n + k) * h_i + i) * w_i + j] = v;
        }
    }
}

__global__ void kcrs_to_ckq_kernel(const float *__restrict__ w, int k_n, int c_n,
                                   float4 *__restrict__ out) {
    int64_t total = (int64_t)c_n * 3 * k_n;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        int k = (int)(t % k_n);
        int64_t r = t / k_n;
        int kh = (int)(r % 3);
        int c = (int)(r / 3);
        const float *src = w + (((int64_t)k * c_n + c) * 3 + kh) * 3;  // [K][C][3][3] row kh
        out[t] = make_float4(src[0], src[1], src[2], 0.0f);
    }
}

}  // namespace
}  // namespace fscnn

using namespace fscnn;

extern "C" {

int fscnn_si_pack3x3(const float *w_kc33, int k, int c, float *wq, void *stream) {
    FSCNN_REQUIRE(k > 0 && c > 0 && w_kc33 && wq, "bad SI pack arguments");
    int64_t total = (int64_t)c * 3 * k;
    unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    kcrs_to_ckq_kernel<<<blocks, 256, 0, as_stream(stream)>>>(w_kc33, k, c,
                                                              reinterpret_cast<float4 *>(wq));
    FSCNN_LAUNCH_CHECK("kcrs_to_ckq_kernel");
    return FSCNN_OK;
}

int fscnn_si_conv3x3(const fscnn_node *in_nodes, const int64_t *in_seg_off, int n, int c, int h,
                     int w, const float *wq, int k, const float *bias, float *y, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0, "bad extents");
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(in_nodes && in_seg_off && wq && y, "null buffer");
    // Strip width: 8 outputs per warp reuse each node for up to three of them, but a
    // small problem (one image, as the per-image layer API runs) then fills only a few
    // SMs; halve the strip until about 24 warps per SM are busy (2 outputs minimum).
    const int64_t k_blocks = ceil_div(k, 32);
    auto warps_for = [&](int s_) { return (int64_t)n * h * ceil_div(w, s_) * k_blocks; };
    const int S = warps_for(8) >= 148 * 24 ? 8 : (warps_for(4) >= 148 * 24 ? 4 : 2);
    const int strips = (int)ceil_div(w, S);
    const size_t ws_bytes = (size_t)c * 3 * 32 * sizeof(float4);
    // Shared-memory weights pay off when two 512-thread CTAs still fit per SM (C <= 66)
    // or when the problem is too small to fill the GPU anyway (one image, e.g. config 2:
    // 43 -> 23 us); for C = 128 at batch 32 the halved occupancy costs more than the
    // L2 weight traffic it saves (measured, tools/prof_si.py).
    const bool small = warps_for(S) < 148 * 24;
    if (ws_bytes <= 200 * 1024 && (ws_bytes <= 100 * 1024 || small) && getenv("FSCNN_SI_NOSMEM") == nullptr) {
        // shallow bank: weights in shared memory, persistent CTAs (1 or 2 per SM)
        const int per_sm = ws_bytes <= 100 * 1024 ? 2 : 1;
        const int64_t jobs = (int64_t)n * h * strips;
        // one-image problems: one CTA per SM over all filter blocks (jobs dealt
        // round-robin), fewer when there are not ~4 jobs per CTA
        const int64_t ctas = std::max<int64_t>(1, std::min<int64_t>(ceil_div(148 * per_sm, k_blocks),
                                                                    ceil_div(jobs, small ? 4 : 16)));
        dim3 g2((unsigned)ctas, (unsigned)k_blocks, 1);
        auto launch = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ws_bytes);
            kern<<<g2, 512, ws_bytes, as_stream(stream)>>>(reinterpret_cast<const int2 *>(in_nodes), in_seg_off,
                                                          n, c, h, w, reinterpret_cast<const float4 *>(wq), k,
                                                          strips, bias, y);
        };
        // one-image problems (config 2): the fiber walks' L2 latency is exposed, so read
        // fibers 32 nodes per coalesced load (walk_fiber COOP)
        if (small) {
            if (S == 8) launch(si_strip_smem_kernel<8, true>);
            else if (S == 4) launch(si_strip_smem_kernel<4, true>);
            else launch(si_strip_smem_kernel<2, true>);
        } else {
            if (S == 8) launch(si_strip_smem_kernel<8, false>);
            else if (S == 4) launch(si_strip_smem_kernel<4, false>);
            else launch(si_strip_smem_kernel<2, false>);
        }
        FSCNN_LAUNCH_CHECK("si_strip_smem_kernel");
        return FSCNN_OK;
    }
    dim3 grid((unsigned)ceil_div((int64_t)h * strips, 4), (unsigned)k_blocks, (unsigned)n);
    auto args = [&](auto kern) {
        kern<<<grid, 128, 0, as_stream(stream)>>>(reinterpret_cast<const int2 *>(in_nodes), in_seg_off, c,
                                                   h, w, reinterpret_cast<const float4 *>(wq), k, strips,
                                                   bias, y);
    };
    if (S == 8) args(si_strip_kernel<8>);
    else if (S == 4) args(si_strip_kernel<4>);
    else args(si_strip_kernel<2>);
    FSCNN_LAUNCH_CHECK("si_strip_kernel");
    return FSCNN_OK;
}

int fscnn_si_conv(const fscnn_node *in_nodes, const int64_t *in_seg_off, int n, int c, int h,
                  int w, const float *wt, int k, int h_f, int w_f, int stride, int pad,
                  const float *bias, float *y, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0, "bad extents");
    FSCNN_REQUIRE(h_f > 0 && w_f > 0 && stride > 0 && pad >= 0, "bad geometry");
    FSCNN_REQUIRE(h_f <= h + 2 * pad && w_f <= w + 2 * pad, "filter exceeds padded input");
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(in_nodes && in_seg_off && wt && y, "null buffer");
    int n_h = (h + 2 * pad - h_f) / stride + 1;
    int n_w = (w + 2 * pad - w_f) / stride + 1;
    dim3 grid((unsigned)ceil_div((int64_t)n_h * n_w, kPixPerBlock), (unsigned)ceil_div(k, 32),
              (unsigned)n);
    si_gather_kernel<<<grid, kPixPerBlock * 32, 0, as_stream(stream)>>>(
        reinterpret_cast<const int2 *>(in_nodes), in_seg_off, c, h, w, wt, k, h_f, w_f, stride,
        pad, n_h, n_w, bias, y);
    FSCNN_LAUNCH_CHECK("si_gather_kernel");
    return FSCNN_OK;
}

}  // extern "C"
