// Sparse-Input 3x3 / stride 1 / pad 1 convolution, channel-major (the fast path).
//
// Same contraction as _conv_input_sparse_kernel (kernels.py:136-166) over the
// reference's CHW input node format, but summed channel by channel instead of in the
// reference's per-output tap-major order, so results agree with the reference to fp32
// reassociation (north star: max|err| <= 1e-4 max|ref|), not bit for bit; the
// bit-exact kernels are si_conv.cu's.
//
// Why a second kernel: the reference order pins every output's running sum to one
// tap-major walk, so the exact kernels fetch a weight line per (node, output row) and
// are bound by that weight stream (16 B of weights per 3 FMAs per lane).  Here the
// order is free, so each weight is loaded once per (CTA, channel) into registers and
// reused for every nonzero input of that channel in the tile:
//   * a warp owns a 4 x 8 output tile of one image and 32*KT filters (lane = filter;
//     KT = 2 from K = 128 up: the accumulator of an output is the register pair of two
//     filters and every FMA an FFMA2 with the input value broadcast); a CTA's NW warps
//     cover up to 512 filters of the same tile.
//   * per 32-channel chunk the CTA decodes the 6 x 10 input region's node fibers into
//     shared memory: values [32][region] plus, per channel, a bitmap of the region
//     positions holding a node (each fiber read as one coalesced 32-node warp load,
//     cursors kept across chunks; 8-warp CTAs prefetch the next chunk's windows with
//     cp.async), then compacts the bitmaps into per-channel entry lists {pos, value}.
//   * each warp walks the chunk's live channels (ascending) and, per channel, its
//     entries (positions ascending): one jump-table branch per entry selects a block of
//     <= 9 FMAs with compile-time accumulator and weight registers (si3x3_cases.inc).
//     The next channel's weights are fetched while the current channel is applied.
// No global atomics; the summation order is fixed, so results are deterministic and
// independent of the batch, KT and the CTA size.
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"

namespace fscnn {
namespace {

#include "si3x3_cases.inc"

constexpr int kSiCC = 32;  // channels per shared-memory chunk

template <int KT> struct SiAcc;
template <> struct SiAcc<1> { using T = float; };
template <> struct SiAcc<2> { using T = unsigned long long; };  // (filter f0, filter f1)

// KT filters per lane (lane l of warp w owns filters (w*KT + j)*32 + l, j < KT).
template <int TY, int TX, int NW, int KT>
__global__ void __launch_bounds__(NW * 32, (TY * TX * KT <= 48 ? 24 : 16) / NW)
    si3x3_fast_kernel(const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off,
                      int64_t n_nodes, int c_n, int h, int w, const float *__restrict__ wf, int k_n,
                      int kp, int tiles_x, const float *__restrict__ bias, float *__restrict__ y,
                      int pool) {
    using AccT = typename SiAcc<KT>::T;
    constexpr int RY = TY + 2, RX = TX + 2, NP = RY * RX, NWD = (NP + 31) / 32;
    __shared__ float val[kSiCC][NP];
    __shared__ unsigned msk[kSiCC][NWD];
    __shared__ int2 ents[kSiCC * (NP + 1) + 1];  // {pos, value} per channel + sentinel {NP, 0},
                                                // + one slot the loop's look-ahead may read
    __shared__ int ch_off[kSiCC + 1];
    __shared__ unsigned ch_live;  // chunk channels with at least one node in the region
    __shared__ int64_t cur[NP];
    // the next chunk's 32-node window of every fiber (cp.async), 8-warp CTAs only: the
    // smaller CTAs are occupancy-bound and load the windows directly
    constexpr bool kStage = NW == 8;
    __shared__ int2 stg[kStage ? NP : 1][32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ty0 = (blockIdx.x / tiles_x) * TY, tx0 = (blockIdx.x % tiles_x) * TX;
    const int img = blockIdx.z;
    const int grp = blockIdx.y * NW + warp;  // this warp's block of 32*KT filters
    for (int p = threadIdx.x; p < NP; p += NW * 32) {
        const int yy = ty0 - 1 + p / RX, xx = tx0 - 1 + p % RX;
        cur[p] = (yy >= 0 && yy < h && xx >= 0 && xx < w) ? seg_off[((int64_t)img * w + xx) * h + yy] : -1;
    }
    AccT acc[TY * TX];
#pragma unroll
    for (int i = 0; i < TY * TX; ++i) acc[i] = AccT(0);
    // bank [C][Kp/(32 KT)][9][32] of AccT: one block of 9 x 32 AccT per (channel, group)
    const AccT *wk = reinterpret_cast<const AccT *>(wf) + (int64_t)grp * 288 + lane;
    const int64_t ch_stride = (int64_t)(kp / (32 * KT)) * 288;
    const uint32_t ents_base = (uint32_t)__cvta_generic_to_shared(ents);
    // Fiber windows are fetched one chunk ahead with cp.async, so the decode reads
    // shared memory; positions outside the image / past the node buffer read sentinels.
    auto fetch = [&](int p, int64_t q) {
        if constexpr (!kStage) return;
        int2 *dst = &stg[kStage ? p : 0][lane];
        if (q >= 0 && q + lane < n_nodes) {
            const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(nodes + q + lane) : "memory");
        } else {
            *dst = make_int2(-1, 0);
        }
    };
    __syncthreads();  // cur[] initialised
    for (int p = warp; p < NP; p += NW) fetch(p, cur[p]);
    asm volatile("cp.async.commit_group;" ::: "memory");

    for (int c0 = 0; c0 < c_n; c0 += kSiCC) {
        for (int i = threadIdx.x; i < kSiCC * NWD; i += NW * 32) (&msk[0][0])[i] = 0u;
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();  // previous chunk applied, masks cleared, windows landed
        // 1. decode: one warp per region position, its staged 32-node window
        const int cend = c0 + kSiCC;
        for (int p = warp; p < NP; p += NW) {
            const int64_t q = cur[p];
            if (q < 0) continue;
            int2 nd = make_int2(-1, 0);
            if constexpr (kStage)
                nd = stg[p][lane];
            else if (q + lane < n_nodes)
                nd = nodes[q + lane];
            const unsigned stop = __ballot_sync(0xffffffffu, nd.x < 0 || nd.x >= cend);
            const int t = stop ? __ffs(stop) - 1 : 32;
            if (lane < t) {
                const int cl = nd.x - c0;
                val[cl][p] = __int_as_float(nd.y);
                atomicOr(&msk[cl][p >> 5], 1u << (p & 31));
            }
            __syncwarp();
            if (lane == 0) cur[p] = q + t;
            if (cend < c_n) fetch(p, q + t);  // the next chunk's window
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        __syncthreads();
        // 2. per-channel entry lists, positions ascending, each closed by a sentinel
        if (warp == 0) {
            int cnt = 0;
#pragma unroll
            for (int j = 0; j < NWD; ++j) cnt += __popc(msk[lane][j]);
            cnt += cnt ? 1 : 0;
            int inc = cnt;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            ch_off[lane] = inc - cnt;
            if (lane == 31) ch_off[kSiCC] = inc;
            const unsigned live = __ballot_sync(0xffffffffu, cnt > 0);
            if (lane == 0) ch_live = live;
        }
        __syncthreads();
        for (int cl = warp; cl < kSiCC; cl += NW) {
            int base = ch_off[cl];
#pragma unroll
            for (int j = 0; j < NWD; ++j) {
                const unsigned m = msk[cl][j];
                const int pos = j * 32 + lane;
                if ((m >> lane) & 1u)
                    ents[base + __popc(m & ((1u << lane) - 1u))] = make_int2(pos, __float_as_int(val[cl][pos]));
                base += __popc(m);
            }
            if (lane == 0 && base > ch_off[cl]) ents[base] = make_int2(NP, 0);
        }
        __syncthreads();
        // 3. apply: channels ascending, each with its 9 weights (per filter) in registers
        unsigned cm = ch_live;
        if (cm == 0u) continue;
        int c = __ffs(cm) - 1;
        // (ping-ponging two weight register sets instead of copying measured 10 % slower:
        // the second copy of the position code costs more in instruction fetch)
        AccT wc[9];
        {
            const AccT *src = wk + (c0 + c) * ch_stride;
#pragma unroll
            for (int t = 0; t < 9; ++t) wc[t] = __ldg(src + t * 32);
        }
        while (true) {
            cm &= cm - 1u;
            const int cn = cm ? __ffs(cm) - 1 : c;
            AccT wn[9];  // the next live channel's weights, in flight during this one
            {
                const AccT *src = wk + (c0 + cn) * ch_stride;
#pragma unroll
                for (int t = 0; t < 9; ++t) wn[t] = __ldg(src + t * 32);
            }
            if constexpr (KT == 1)
                si_chan<TY, TX>(acc, wc, ents_base + 8u * (uint32_t)ch_off[c]);
            else
                si_chan2<TY, TX>(acc, wc, ents_base + 8u * (uint32_t)ch_off[c]);
            if (cm == 0u) break;
            c = cn;
#pragma unroll
            for (int t = 0; t < 9; ++t) wc[t] = wn[t];
        }
    }
    if (pool) {
        // Alg. 7 (layers.py:345-390): the conv output pooled 2x2 inside the tile (tiles
        // sit at even coordinates), in pool2d's order -- (ph, pw) row-major, max from
        // -inf with '>', avg as a left-to-right sum (first NaN wins) / 4 -- then + bias
        const int ho = h >> 1, wo = w >> 1;
#pragma unroll
        for (int j = 0; j < KT; ++j) {
            const int k = (grp * KT + j) * 32 + lane;
            if (k >= k_n) continue;
            const float bk = bias ? bias[k] : 0.0f;
            float *yk = y + ((int64_t)img * k_n + k) * ho * wo;
#pragma unroll
            for (int qy = 0; qy < TY / 2; ++qy) {
                const int yy = (ty0 >> 1) + qy;
                if (yy >= ho) break;
#pragma unroll
                for (int qx = 0; qx < TX / 2; ++qx) {
                    const int xx = (tx0 >> 1) + qx;
                    if (xx >= wo) break;
                    float m = pool == 1 ? -INFINITY : 0.0f;
#pragma unroll
                    for (int ph = 0; ph < 2; ++ph)
#pragma unroll
                        for (int pw = 0; pw < 2; ++pw) {
                            const int o = (2 * qy + ph) * TX + 2 * qx + pw;
                            float v;
                            if constexpr (KT == 1)
                                v = acc[o];
                            else
                                v = __uint_as_float((unsigned)(acc[o] >> (32 * j)));
                            v = (v != 0.0f) ? v : 0.0f;
                            if (pool == 1) {
                                if (v > m) m = v;
                            } else if (!is_nan_bits(m)) {
                                m = is_nan_bits(v) ? nan_quiet(v) : __fadd_rn(m, v);
                            }
                        }
                    if (pool == 2 && !is_nan_bits(m)) m = __fdiv_rn(m, 4.0f);
                    if (bias) m = __fadd_rn(m, bk);
                    yk[(int64_t)yy * wo + xx] = m;
                }
            }
        }
        return;
    }
#pragma unroll
    for (int j = 0; j < KT; ++j) {
        const int k = (grp * KT + j) * 32 + lane;
        if (k >= k_n) continue;
        const float bk = bias ? bias[k] : 0.0f;
        float *yk = y + ((int64_t)img * k_n + k) * h * w;
#pragma unroll
        for (int oy = 0; oy < TY; ++oy) {
            const int yy = ty0 + oy;
            if (yy >= h) break;
#pragma unroll
            for (int ox = 0; ox < TX; ++ox) {
                const int xx = tx0 + ox;
                if (xx >= w) break;
                float v;
                if constexpr (KT == 1)
                    v = acc[oy * TX + ox];
                else
                    v = __uint_as_float((unsigned)(acc[oy * TX + ox] >> (32 * j)));
                v = (v != 0.0f) ? v : 0.0f;  // a zero sum is +0.0 (no node in the reference)
                if (bias) v = __fadd_rn(v, bk);
                yk[(int64_t)yy * w + xx] = v;
            }
        }
    }
}

// Launch geometry for a layer of K filters; the bank layout depends on it.  KT filters
// per lane, NW warps per CTA, and Kp = K padded with zero filters to whole CTAs (every
// warp of the grid owns real bank rows).
struct SiGeom {
    int kt, nw, kp;
};
inline SiGeom si_fast_geom(int k) {
    SiGeom g;
    g.kt = k >= 128 ? 2 : 1;
    const int groups = (int)ceil_div(k, 32 * g.kt);
    g.nw = groups >= 8 ? 8 : (groups >= 4 ? 4 : 2);
    g.kp = (int)ceil_div(k, 32 * g.kt * g.nw) * 32 * g.kt * g.nw;
    return g;
}

// [K][C][3][3] -> [C][Kp/(32 KT)][9][32][KT] (tap = kh*3 + kw; zero past K)
__global__ void si_pack_fast_kernel(const float *__restrict__ w, int k_n, int c_n, int kp, int kt,
                                    float *__restrict__ out) {
    const int64_t total = (int64_t)c_n * 9 * kp;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int ng = kp / (32 * kt);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += stride) {
        const int j = (int)(t % kt);
        const int64_t r0 = t / kt;
        const int lane = (int)(r0 & 31);
        const int64_t r = r0 >> 5;
        const int tap = (int)(r % 9);
        const int64_t r2 = r / 9;
        const int g = (int)(r2 % ng), c = (int)(r2 / ng);
        const int k = (g * kt + j) * 32 + lane;
        out[t] = k < k_n ? w[((int64_t)k * c_n + c) * 9 + tap] : 0.0f;
    }
}

template <int TY, int TX, int NW, int KT>
int launch_fast(const int2 *nodes, const int64_t *seg_off, int64_t n_nodes, int n, int c, int h, int w,
                const float *wf, int k, int kp, const float *bias, float *y, cudaStream_t st, int pool) {
    const int tiles_x = (int)ceil_div(w, TX), tiles_y = (int)ceil_div(h, TY);
    dim3 grid((unsigned)(tiles_x * tiles_y), (unsigned)ceil_div(kp, NW * 32 * KT), (unsigned)n);
    si3x3_fast_kernel<TY, TX, NW, KT><<<grid, NW * 32, 0, st>>>(nodes, seg_off, n_nodes, c, h, w, wf, k, kp,
                                                                tiles_x, bias, y, pool);
    FSCNN_LAUNCH_CHECK("si3x3_fast_kernel");
    return FSCNN_OK;
}

}  // namespace
}  // namespace fscnn

using namespace fscnn;

extern "C" {

int64_t fscnn_si_fast_bank_floats(int k, int c) {
    if (k <= 0 || c <= 0) return 0;
    return (int64_t)c * 9 * si_fast_geom(k).kp;
}

int fscnn_si_pack_fast(const float *w_kc33, int k, int c, float *wf, void *stream) {
    FSCNN_REQUIRE(k > 0 && c > 0 && w_kc33 && wf, "bad SI pack arguments");
    const SiGeom g = si_fast_geom(k);
    const int64_t total = (int64_t)c * 9 * g.kp;
    const unsigned blocks = (unsigned)std::min<int64_t>(ceil_div(total, 256), 148 * 16);
    si_pack_fast_kernel<<<blocks, 256, 0, as_stream(stream)>>>(w_kc33, k, c, g.kp, g.kt, wf);
    FSCNN_LAUNCH_CHECK("si_pack_fast_kernel");
    return FSCNN_OK;
}

int fscnn_si_conv3x3_fast_pool(const fscnn_node *in_nodes, const int64_t *in_seg_off, int64_t n_nodes, int n,
                               int c, int h, int w, const float *wf, int k, const float *bias, int pool,
                               float *y, void *stream) {
    FSCNN_REQUIRE(pool >= 0 && pool <= 2, "pool must be 0 (none), 1 (2x2 max) or 2 (2x2 avg)");
    if (pool) FSCNN_REQUIRE(h % 2 == 0 && w % 2 == 0, "fused 2x2 pool needs even extents");
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0 && n_nodes >= 0, "bad extents");
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(in_nodes && in_seg_off && wf && y, "null buffer");
    FSCNN_REQUIRE(n <= 65535, "batch too large for one launch (%d > 65535)", n);
    const SiGeom g = si_fast_geom(k);
    const int kt = g.kt, nw = g.nw, kp = g.kp;
    const int2 *nd = reinterpret_cast<const int2 *>(in_nodes);
    cudaStream_t st = as_stream(stream);
    if (kt == 2) {
        if (nw == 8) return launch_fast<4, 8, 8, 2>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
        if (nw == 4) return launch_fast<4, 8, 4, 2>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
        return launch_fast<4, 8, 2, 2>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
    }
    // one filter per lane (K < 128)
    if (nw == 8) return launch_fast<4, 8, 8, 1>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
    if (nw == 4) return launch_fast<4, 8, 4, 1>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
    return launch_fast<4, 8, 2, 1>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, kp, bias, y, st, pool);
}

int fscnn_si_conv3x3_fast(const fscnn_node *in_nodes, const int64_t *in_seg_off, int64_t n_nodes, int n,
                          int c, int h, int w, const float *wf, int k, const float *bias, float *y,
                          void *stream) {
    return fscnn_si_conv3x3_fast_pool(in_nodes, in_seg_off, n_nodes, n, c, h, w, wf, k, bias, 0, y, stream);
}

}  // extern "C"
