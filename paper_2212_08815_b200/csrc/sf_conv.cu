// Sparse-Filter convolution kernels.
//
// 1) sf_exact_kernel -- reference accumulation order, bit-exact with
//    _conv_all_filters_kernel (layers.py:170-180) / _window_acc (kernels.py:78-97):
//    one thread per output pixel, warp-uniform filter k; taps kw outer, kh inner,
//    nodes ascending c; __fmul_rn + __fadd_rn (no contraction, like numba).
//    Any geometry.  Reads the reference's CHW node buffer directly.
//
// 2) sf3x3_kernel -- the fast path for 3x3/s1/p1 (all VGG16 convs).  Dense activations x
//    unstructured-sparse filters on FP32 CUDA cores:
//      * a CTA owns 32 lane tiles (LI sub-regions of (4*LY) x 16 output pixels, LY*LI = 8)
//        and 32 output channels; warp w owns filter group g (KT = 4 filters);
//      * lane = one 4x4 output tile; acc[KT][4][4] in registers as FFMA2 column pairs;
//      * input channels stream through shared memory in chunks of CC channels: one TMA
//        box per sub-region per chunk ((4LY+2) x 20 floats x CC, zero fill for the conv
//        padding) plus a bulk copy of each warp's packed nonzero list, completed on an
//        mbarrier (S-stage ring).  No producer warp: each warp restages its own entry
//        run as soon as it leaves a stage, and the last warp to leave (smem counter)
//        restages the shared boxes, so warps drift freely within the ring;
//      * per channel a lane loads its 6x6 input patch into registers, then walks the
//        warp-uniform nonzero list through a jump table (sf3x3_dispatch.inc, generated
//        by gen_sf3x3_dispatch.py): each nonzero is 8 FFMA2 / 16 FFMA on statically
//        named registers, every loaded input value reused by all nonzeros of the channel;
//      * epilogue: + bias, optional ReLU, optional fused 2x2 max-pool (the reference's
//        relu -> pool order, -inf start, '>' compare).
#include <cuda.h>
#include <stdlib.h>

#include "common.cuh"
#include "sf3x3_dispatch.inc"

namespace fscnn {
namespace {

// ------------------------------------------------------------------------------
// exact, reference-order kernel
// ------------------------------------------------------------------------------
__global__ void sf_exact_kernel(const float *__restrict__ x, int c_n, int h_i, int w_i,
                                const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off,
                                int k_n, int h_f, int w_f, int stride, int pad, int n_h, int n_w,
                                const float *__restrict__ bias, int relu, float *__restrict__ y) {
    int k = blockIdx.y;
    int img = blockIdx.z;
    int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= n_h * n_w) return;
    int i = pix / n_w, j = pix % n_w;
    const float *xi = x + (int64_t)img * c_n * h_i * w_i;
    int64_t seg_base = (int64_t)k * h_f * w_f;
    float acc = 0.0f;
    for (int l = 0; l < w_f; ++l) {
        int w_in = l + j * stride - pad;
        if (w_in < 0 || w_in >= w_i) continue;
        for (int kk = 0; kk < h_f; ++kk) {
            int h_in = kk + i * stride - pad;
            if (h_in < 0 || h_in >= h_i) continue;
            const float *px = xi + (int64_t)h_in * w_i + w_in;
            int64_t p = seg_off[seg_base + (int64_t)l * h_f + kk];
            for (int2 nd = nodes[p]; nd.x != -1; nd = nodes[++p])
                acc = __fadd_rn(acc, __fmul_rn(px[(int64_t)nd.x * h_i * w_i], __int_as_float(nd.y)));
        }
    }
    float b = bias ? bias[k] : 0.0f;
    float v = __fadd_rn(acc, b);
    if (relu) v = relu_np(v);
    y[(((int64_t)img * k_n + k) * n_h + i) * n_w + j] = v;
}

// Dense baseline conv (conv_forward_dense, layers.py:326-342, over _dense_conv_kernel
// kernels.py:169-192): taps kh outer, kw inner, channels ascending, every weight
// (zeros included) multiplied as inp * filt, then + bias -- bit-exact with numba.
// Same thread mapping as sf_exact_kernel; wt is the dense [K][C][h_f][w_f] bank.
__global__ void dense_exact_kernel(const float *__restrict__ x, int c_n, int h_i, int w_i,
                                   const float *__restrict__ wt, int k_n, int h_f, int w_f,
                                   int stride, int pad, int n_h, int n_w,
                                   const float *__restrict__ bias, float *__restrict__ y) {
    int k = blockIdx.y;
    int img = blockIdx.z;
    int pix = blockIdx.x * blockDim.x + threadIdx.x;
    if (pix >= n_h * n_w) return;
    int i = pix / n_w, j = pix % n_w;
    const int64_t plane = (int64_t)h_i * w_i;
    const float *xi = x + (int64_t)img * c_n * plane;
    const float *wk = wt + (int64_t)k * c_n * h_f * w_f;
    float acc = 0.0f;
    for (int kk = 0; kk < h_f; ++kk) {
        int h_in = kk + i * stride - pad;
        if (h_in < 0 || h_in >= h_i) continue;
        for (int l = 0; l < w_f; ++l) {
            int w_in = l + j * stride - pad;
            if (w_in < 0 || w_in >= w_i) continue;
            const float *px = xi + (int64_t)h_in * w_i + w_in;
            const float *pw = wk + kk * w_f + l;
            for (int c = 0; c < c_n; ++c)
                acc = __fadd_rn(acc, __fmul_rn(px[c * plane], pw[(int64_t)c * h_f * w_f]));
        }
    }
    y[(((int64_t)img * k_n + k) * n_h + i) * n_w + j] = __fadd_rn(acc, bias ? bias[k] : 0.0f);
}

// ------------------------------------------------------------------------------
// fast 3x3 kernel
// ------------------------------------------------------------------------------
// KT filters per warp (1, 2, 4 or 8, == the pack's kt); a CTA holds 32 filters for KT = 4
// (8 warps, <=128 regs, 2 CTAs = 16 warps/SM) and 8 (4 warps), 16 for KT = 2 (8 warps)
// and 4 for KT = 1 (4 warps): more CTAs and shorter dispatch chains per warp for layers
// whose KT = 4 grid cannot fill the GPU (small batches).  Each filter's accumulation
// order (channels ascending, then its taps ascending) does not depend on KT or the CTA
// size, so the results are bit-identical.
#ifndef FSCNN_SF3_CTA_FILTERS
#define FSCNN_SF3_CTA_FILTERS 32
#endif
constexpr int CTA_FILTERS = FSCNN_SF3_CTA_FILTERS;
constexpr int CTAS_PER_SM = CTA_FILTERS == 32 ? 2 : 1;
// Default warps per CTA for KT; a launch may ask for 4-warp CTAs with KT = 2 (8 filters
// per CTA) when even the 16-filter grid leaves most SMs idle.
template <int KT> struct SfCfg {
    static constexpr int NWARP = KT <= 2 ? (KT == 2 ? 8 : 4) : CTA_FILTERS / KT;
};
constexpr int MAX_STAGES = 4;
constexpr int BOXW = 20;           // smem row pitch (floats) == TMA box width
constexpr int TILE = 4;            // lane tile is TILE x TILE outputs
constexpr int SUBW = 16;           // sub-region width (4 lanes x 4 columns)


__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// The value of lane 0 through redux.sync, which ptxas knows to be warp-uniform (it lands
// in a uniform register).  Used for the entry cursor: when ptxas cannot prove the jump
// index uniform it guards the jump-table loop with a per-nonzero convergence barrier
// (BSSY/BSYNC + an extra branch per nonzero).
__device__ __forceinline__ uint32_t warp_uniform(uint32_t v) {
    uint32_t r;
    asm volatile("redux.sync.min.u32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(v));
    return r;
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(addr),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void tma_load_4d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0,
                                            int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void bulk_load(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

struct Sf3Params {
    const int2 *packed;       // packed filter stream (+16 B slack at the end)
    const int64_t *seg_off;   // [groups][C] segment offsets
    int64_t total_nodes;      // length of packed
    int n, c, h, w;           // input extents (NCHW, row pitch = TMA stride)
    int k;                    // output channels
    int ldo;                  // output row pitch (floats)
    int tiles_h, tiles_w;     // sub-region grid per image
    int n_sub;                // n * tiles_h * tiles_w
    int n_fb;                 // filter blocks (CTA_FILTERS filters each)
    int cc;                   // channels per chunk
    int ent_cap;              // entry slots per warp per stage (int2)
    int box_floats;           // floats per sub-region box per stage
    const float *bias;
    float *y;
    int relu;
    int pool;                 // fused 2x2 max-pool
    int stages;               // ring depth (<= MAX_STAGES)
    int dbg;                  // debug (FSCNN_SF3_DEBUG, wrong results): 5 = no box TMA;
                              // 7 = entries restaged per warp, boxes never restaged;
                              // 8 = no epilogue stores
};

template <int LY, int KT, int NW>
__global__ void __launch_bounds__(NW * 32, CTAS_PER_SM)
    sf3x3_kernel(const __grid_constant__ CUtensorMap tmap, const Sf3Params p) {
    constexpr int NWARP = NW;
    constexpr int NTHREADS = NW * 32;
    constexpr int LI = 8 / LY;          // sub-regions per CTA
    constexpr int SUBH = TILE * LY;     // sub-region height
    constexpr int BOXH = SUBH + 2;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    float *in_s = reinterpret_cast<float *>(smem_raw);
    const int STAGES = p.stages;
    const int stage_in_floats = LI * p.box_floats;
    int2 *ent_s = reinterpret_cast<int2 *>(in_s + STAGES * stage_in_floats);
    uint64_t *full = reinterpret_cast<uint64_t *>(ent_s + STAGES * NWARP * p.ent_cap);
    int *done = reinterpret_cast<int *>(full + STAGES);    // per-stage finished-warp counters
    int *cofs = done + 2 * STAGES;                           // [NWARP][n_chunks + 1] run starts

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // 1-D grid, filter block fastest: the CTAs of one spatial unit (all filter blocks)
    // run together, so its input boxes are read from DRAM once and then hit in L2
    const int n_fb = p.n_fb;
    const int sub0 = (int)(blockIdx.x / n_fb) * LI;
    const int g0 = (int)(blockIdx.x % n_fb) * NWARP;
    const int n_groups = (p.k + KT - 1) / KT;
    const int n_chunks = (p.c + p.cc - 1) / p.cc;

    // chunk-run table: cofs[w][j] = first packed node of group g0+w, channel j*cc
    // (j = n_chunks: one past the group's last node) -- keeps global loads off the loop
    for (int idx = threadIdx.x; idx < NWARP * (n_chunks + 1); idx += NTHREADS) {
        const int wv = idx / (n_chunks + 1), j = idx % (n_chunks + 1);
        const int gg = g0 + wv;
        int64_t v = 0;
        if (gg < n_groups) {
            if (j < n_chunks) v = p.seg_off[(int64_t)gg * p.c + (int64_t)j * p.cc];
            else v = (gg + 1 < n_groups) ? p.seg_off[(int64_t)(gg + 1) * p.c] : p.total_nodes;
        }
        cofs[idx] = (int)v;
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            // NWARP entry-run arrivals + 1 input-box arrival complete a stage
            mbar_init(&full[s], NWARP + 1);
            done[s] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmap)) : "memory");
    }
    __syncthreads();

    const int g = g0 + warp;
    const bool live = g < n_groups;
    int n_box = 0;
#pragma unroll
    for (int li = 0; li < LI; ++li) n_box += (sub0 + li < p.n_sub);
    const uint32_t box_bytes =
        p.dbg == 5 ? 0u : (uint32_t)n_box * (uint32_t)(BOXW * BOXH * p.cc * 4);

    // Each warp stages its own entry run for chunk ch (lane 0); dead groups arrive empty.
    auto refill_entries = [&](int ch) {
        const int s = ch % STAGES;
        uint32_t nb = 0;
        int lo = 0;
        if (live) {
            const int a = cofs[warp * (n_chunks + 1) + ch];
            const int b = cofs[warp * (n_chunks + 1) + ch + 1];
            lo = a & ~1;  // 16-byte aligned start
            nb = (uint32_t)(((b - lo) * 8 + 15) & ~15);
        }
        mbar_expect_tx(&full[s], nb);
        if (nb) bulk_load(ent_s + (s * NWARP + warp) * p.ent_cap, p.packed + lo, nb, &full[s]);
    };
    // The shared input boxes of chunk ch (the TMA zero-fills the conv padding).
    auto refill_boxes = [&](int ch) {
        const int s = ch % STAGES;
        mbar_expect_tx(&full[s], box_bytes);
        if (p.dbg == 5) return;
#pragma unroll
        for (int li = 0; li < LI; ++li) {
            int sub = sub0 + li;
            if (sub >= p.n_sub) continue;
            int tw = sub % p.tiles_w;
            int r = sub / p.tiles_w;
            int th = r % p.tiles_h;
            int img = r / p.tiles_h;
            // rows th*SUBH-1 .. +SUBH and logical cols tw*SUBW-1 .. +18 = memory cols
            // tw*SUBW .. +19 of the halo-column layout (16-byte aligned innermost start:
            // the TMA unit faults on a misaligned one)
            tma_load_4d(in_s + s * stage_in_floats + li * p.box_floats, &tmap, &full[s],
                        tw * SUBW, th * SUBH - 1, ch * p.cc, img);
        }
    };

    // A dead group (k not a multiple of the CTA's filters) walks "empty channel"
    // markers, so the dispatch call needs no enclosing branch.
    if (!live)
        for (int i = lane; i < STAGES * p.ent_cap; i += 32)
            ent_s[((i / p.ent_cap) * NWARP + warp) * p.ent_cap + i % p.ent_cap] =
                make_int2(2 * KT * 9, 0x7fffffff);  // one run covering the whole chunk
    if (lane == 0)
        for (int ch = 0; ch < STAGES && ch < n_chunks; ++ch) {
            refill_entries(ch);
            if (warp == 0) refill_boxes(ch);
        }
    __syncwarp();  // the dispatch loop's .uni branches need a converged warp

    const int lx = lane & 3;
    const int ly = (lane >> 2) % LY;
    const int li = lane / (4 * LY);

    // accumulators as column pairs (FFMA2 operands): acc2[kl][py][h] = cols 2h, 2h+1
    unsigned long long acc2[KT][TILE][2];
#pragma unroll
    for (int a = 0; a < KT; ++a)
#pragma unroll
        for (int b = 0; b < TILE; ++b) acc2[a][b][0] = acc2[a][b][1] = 0ull;

#pragma unroll 1
    for (int ch = 0; ch < n_chunks; ++ch) {
        const int s = ch % STAGES;
        mbar_wait(&full[s], (ch / STAGES) & 1);
        __syncwarp();
        const int c0 = ch * p.cc;
        const int cnt = min(p.cc, p.c - c0);
        {
            const int2 *ents = ent_s + (s * NWARP + warp) * p.ent_cap;
            // offset inside the 16-byte aligned copy
            const int e0 = live ? cofs[warp * (n_chunks + 1) + ch] & 1 : 0;
            const float *box = in_s + s * stage_in_floats + li * p.box_floats;
            sf3x3_chunk<BOXW * 4>(acc2, warp_uniform(smem_u32(ents + e0)),
                                  smem_u32(box + (TILE * ly) * BOXW + TILE * lx), cnt,
                                  (uint32_t)(BOXH * BOXW * 4));
        }
        __syncwarp();
        // Stage s is free for this warp: restage its own entry run for chunk ch+STAGES;
        // the last warp to leave the stage also restages the shared input boxes.
        if (lane == 0 && ch + STAGES < n_chunks) {
            refill_entries(ch + STAGES);
            // the counter only grows: every NWARP-th arrival closes a round
            const int prev = atomicAdd(&done[s], 1);
            if (p.dbg == 7) {
                // debug: boxes are never restaged (stale input) and the first warp to
                // leave does the box arrival -- measures the cost of the warp coupling
                if (prev % NWARP == 0) mbar_expect_tx(&full[s], 0);
            } else if ((prev + 1) % NWARP == 0) {
                refill_boxes(ch + STAGES);
            }
        }
        __syncwarp();
    }

    // ---------------- epilogue ----------------
    const int sub = sub0 + li;
    if (g >= n_groups || sub >= p.n_sub) return;
    if (p.dbg == 8) {  // debug: skip the stores (keep the accumulators live)
        float t = 0.0f;
#pragma unroll
        for (int a = 0; a < KT; ++a)
#pragma unroll
            for (int b = 0; b < TILE; ++b) t += __uint_as_float((uint32_t)acc2[a][b][0]);
        if (t == 12345.678f) p.y[0] = t;
        return;
    }
    const int tw = sub % p.tiles_w;
    const int r = sub / p.tiles_w;
    const int th = r % p.tiles_h;
    const int img = r / p.tiles_h;
    const int y0 = th * SUBH + TILE * ly;
    const int x0 = tw * SUBW + TILE * lx;
    if (y0 >= p.h || x0 >= p.w) return;
#pragma unroll
    for (int kl = 0; kl < KT; ++kl) {
        const int k = g * KT + kl;
        if (k >= p.k) break;
        const float b = p.bias ? p.bias[k] : 0.0f;
        float o[TILE][TILE];
#pragma unroll
        for (int py = 0; py < TILE; ++py)
#pragma unroll
            for (int px = 0; px < TILE; ++px) {
                const unsigned long long pr = acc2[kl][py][px >> 1];
                const float a = __uint_as_float((uint32_t)((px & 1) ? (pr >> 32) : (pr & 0xffffffffull)));
                float v = a + b;
                o[py][px] = p.relu ? relu_np(v) : v;
            }
        if (!p.pool) {
            // halo-column layout: logical column x lives at memory column x + 1
            float *dst = p.y + (((int64_t)img * p.k + k) * p.h + y0) * p.ldo + x0 + 1;
            const bool full_row = x0 + TILE <= p.w;
#pragma unroll
            for (int py = 0; py < TILE; ++py) {
                if (y0 + py >= p.h) break;
                float *d = dst + (int64_t)py * p.ldo;
                if (full_row) {
                    // memory columns x0+1 .. x0+4: the middle pair is 8-byte aligned
                    d[0] = o[py][0];
                    *reinterpret_cast<float2 *>(d + 1) = make_float2(o[py][1], o[py][2]);
                    d[3] = o[py][3];
                } else {
#pragma unroll
                    for (int px = 0; px < TILE; ++px)
                        if (x0 + px < p.w) d[px] = o[py][px];
                }
            }
        } else {
            // fused 2x2/2 max-pool: output (h/2, w/2) with row pitch ldo
            const int ho = p.h >> 1, wo = p.w >> 1;
            const int yo0 = y0 >> 1, xo0 = x0 >> 1;
            float *dst = p.y + (((int64_t)img * p.k + k) * ho + yo0) * p.ldo + xo0 + 1;
#pragma unroll
            for (int qy = 0; qy < 2; ++qy) {
                if (yo0 + qy >= ho) break;
#pragma unroll
                for (int qx = 0; qx < 2; ++qx) {
                    if (xo0 + qx >= wo) break;
                    float m = -INFINITY;
#pragma unroll
                    for (int ph = 0; ph < 2; ++ph)
#pragma unroll
                        for (int pw = 0; pw < 2; ++pw) {
                            float v = o[2 * qy + ph][2 * qx + pw];
                            if (v > m) m = v;
                        }
                    dst[(int64_t)qy * p.ldo + qx] = m;
                }
            }
        }
    }
}

// ------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_tiled() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(ptr);
    }
    return fn;
}

template <int LY, int KT, int NW = SfCfg<KT>::NWARP>
int launch_sf3x3(const CUtensorMap &map, Sf3Params &p, cudaStream_t st) {
    constexpr int LI = 8 / LY;
    constexpr int SUBH = TILE * LY;
    p.tiles_h = (int)ceil_div(p.h, SUBH);
    p.tiles_w = (int)ceil_div(p.w, SUBW);
    p.n_sub = p.n * p.tiles_h * p.tiles_w;
    p.box_floats = BOXW * (SUBH + 2) * p.cc;
    // each box must start 128-byte aligned (TMA destination)
    p.box_floats = (p.box_floats + 31) & ~31;
    constexpr int NWARP = NW;
    constexpr int NTHREADS = NW * 32;
    const int n_chunks = (int)ceil_div(p.c, p.cc);
    auto smem_for = [&](int st) {
        return (size_t)st * LI * p.box_floats * 4 + (size_t)st * NWARP * p.ent_cap * 8 + 2 * st * 8 +
               (size_t)NWARP * (n_chunks + 1) * 4;
    };
    // deepest ring that still lets two CTAs share an SM (228 KB, 1 KB reserved each)
    p.stages = MAX_STAGES;
    const size_t budget = CTAS_PER_SM == 2 ? 113 * 1024 : 227 * 1024;
    while (p.stages > 2 && smem_for(p.stages) > budget) --p.stages;
    size_t smem = smem_for(p.stages);
    if (smem > 227 * 1024) {
        set_error("sf3x3: %zu bytes of shared memory needed; lower cc", smem);
        return FSCNN_ERR_UNSUPPORTED;
    }
    auto kern = sf3x3_kernel<LY, KT, NW>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
        set_error("sf3x3: smem attribute (%zu bytes): %s", smem, cudaGetErrorString(e));
        return FSCNN_ERR_CUDA;
    }
    int n_groups = (int)ceil_div(p.k, KT);
    p.n_fb = (int)ceil_div(n_groups, NWARP);
    const int64_t n_cta = ceil_div(p.n_sub, LI) * (int64_t)p.n_fb;
    if (n_cta > 0x7fffffff) {
        set_error("sf3x3: grid of %lld CTAs too large", (long long)n_cta);
        return FSCNN_ERR_UNSUPPORTED;
    }
    dim3 grid((unsigned)n_cta, 1, 1);
    kern<<<grid, NTHREADS, smem, st>>>(map, p);
    return check_launch("sf3x3_kernel");
}

}  // namespace
}  // namespace fscnn

using namespace fscnn;

extern "C" {

int fscnn_sf_conv_exact(const float *x, int n, int c, int h, int w, const fscnn_node *nodes,
                        const int64_t *seg_off, int k, int h_f, int w_f, int stride, int pad,
                        const float *bias, int relu, float *y, void *stream) {
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0, "bad extents");
    FSCNN_REQUIRE(h_f > 0 && w_f > 0 && stride > 0 && pad >= 0, "bad geometry");
    FSCNN_REQUIRE(h_f <= h + 2 * pad && w_f <= w + 2 * pad, "filter exceeds padded input");
    int n_h = (h + 2 * pad - h_f) / stride + 1;
    int n_w = (w + 2 * pad - w_f) / stride + 1;
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && nodes && seg_off && y, "null buffer");
    FSCNN_REQUIRE(k <= 65535 && n <= 65535, "k or n too large for the grid");
    dim3 grid((unsigned)ceil_div((int64_t)n_h * n_w, 128), (unsigned)k, (unsigned)n);
    sf_exact_kernel<<<grid, 128, 0, as_stream(stream)>>>(
        x, c, h, w, reinterpret_cast<const int2 *>(nodes), seg_off, k, h_f, w_f, stride, pad, n_h,
        n_w, bias, relu, y);
    FSCNN_LAUNCH_CHECK("sf_exact_kernel");
    return FSCNN_OK;
}

int fscnn_dense_conv_exact(const float *x, int n, int c, int h, int w, const float *wt, int k,
                           int h_f, int w_f, int stride, int pad, const float *bias, float *y,
                           void *stream) {
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0, "bad extents");
    FSCNN_REQUIRE(h_f > 0 && w_f > 0 && stride > 0 && pad >= 0, "bad geometry");
    FSCNN_REQUIRE(h_f <= h + 2 * pad && w_f <= w + 2 * pad, "filter exceeds padded input");
    int n_h = (h + 2 * pad - h_f) / stride + 1;
    int n_w = (w + 2 * pad - w_f) / stride + 1;
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && wt && y, "null buffer");
    FSCNN_REQUIRE(k <= 65535 && n <= 65535, "k or n too large for the grid");
    dim3 grid((unsigned)ceil_div((int64_t)n_h * n_w, 128), (unsigned)k, (unsigned)n);
    dense_exact_kernel<<<grid, 128, 0, as_stream(stream)>>>(x, c, h, w, wt, k, h_f, w_f, stride, pad,
                                                            n_h, n_w, bias, y);
    FSCNN_LAUNCH_CHECK("dense_exact_kernel");
    return FSCNN_OK;
}

// Extended entry: ldi/ldo are input/output row pitches (floats, multiples of 4);
// pool fuses the 2x2 max-pool; cc/ent_cap/ly are tuning knobs (0 = auto).
int fscnn_sf_conv3x3_ex(const float *x, int n, int c, int h, int w, int ldi,
                        const fscnn_node *packed, const int64_t *packed_seg_off,
                        int64_t total_nodes, int max_chunk_entries, int cc, int k,
                        const float *bias, int relu, int pool, float *y, int ldo, int ly,
                        int kt, void *stream) {
    static const int dbg_mode = getenv("FSCNN_SF3_DEBUG") ? atoi(getenv("FSCNN_SF3_DEBUG")) : 0;
    FSCNN_REQUIRE(n > 0 && c > 0 && h > 0 && w > 0 && k > 0, "bad extents");
    FSCNN_REQUIRE(ldi >= w + 1 && ldi % 4 == 0, "input row pitch must be >= w + 1 and a multiple of 4");
    FSCNN_REQUIRE(ldo >= (pool ? w / 2 : w) + 1, "output row pitch too small");
    // the non-pool epilogue stores a float2 at memory column x0 + 2 of each row
    FSCNN_REQUIRE(ldo % 2 == 0 && (reinterpret_cast<uintptr_t>(y) & 7) == 0,
                  "output row pitch must be even and the output 8-byte aligned");
    FSCNN_REQUIRE(x && packed && packed_seg_off && y, "null buffer");
    FSCNN_REQUIRE(cc > 0 && cc <= 256, "bad channel chunk");
    FSCNN_REQUIRE(max_chunk_entries > 0, "bad entry capacity");
    FSCNN_REQUIRE((reinterpret_cast<uintptr_t>(x) & 15) == 0, "input must be 16-byte aligned");
    if (pool) FSCNN_REQUIRE(h % 2 == 0 && w % 2 == 0, "fused pool needs even extents");
    EncodeTiledFn enc = get_encode_tiled();
    if (!enc) {
        set_error("cuTensorMapEncodeTiled unavailable");
        return FSCNN_ERR_CUDA;
    }
    Sf3Params p{};
    p.packed = reinterpret_cast<const int2 *>(packed);
    p.seg_off = packed_seg_off;
    p.total_nodes = total_nodes;
    p.n = n; p.c = c; p.h = h; p.w = w; p.k = k;
    p.ldo = ldo;
    p.cc = cc;
    // aligned-down start can add one entry, round-up to 16 B another
    p.ent_cap = (max_chunk_entries + 3 + 1) & ~1;
    p.bias = bias; p.y = y; p.relu = relu; p.pool = pool;
    p.dbg = dbg_mode;
    // auto: 16x16 sub-regions (measured fastest on every VGG16 width at 16-channel
    // chunks); 8x16 for very shallow inputs or short images
    if (ly <= 0) ly = (c < 8 || h <= 8) ? 2 : 4;
    int sub_h = TILE * ly;
    CUtensorMap map;
    cuuint64_t gdim[4] = {(cuuint64_t)w + 1, (cuuint64_t)h, (cuuint64_t)c, (cuuint64_t)n};
    cuuint64_t gstride[3] = {(cuuint64_t)ldi * 4, (cuuint64_t)ldi * h * 4,
                             (cuuint64_t)ldi * h * c * 4};
    cuuint32_t box[4] = {(cuuint32_t)BOXW, (cuuint32_t)(sub_h + 2), (cuuint32_t)cc, 1};
    cuuint32_t estride[4] = {1, 1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float *>(x), gdim, gstride,
                     box, estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
        return FSCNN_ERR_CUDA;
    }
    cudaStream_t st = as_stream(stream);
    // kt: filters per warp in the low byte (== the pack's kt); bits 8-15: warps per CTA
    // (0 = default; 4 with kt = 2 for very small grids)
    const int cta_warps = (kt >> 8) & 0xff;
    kt &= 0xff;
    if (kt == 2 && cta_warps == 4) {
        switch (ly) {
            case 8: return launch_sf3x3<8, 2, 4>(map, p, st);
            case 4: return launch_sf3x3<4, 2, 4>(map, p, st);
            case 2: return launch_sf3x3<2, 2, 4>(map, p, st);
            default: break;
        }
    }
    if (kt == 1) {  // 1 filter per warp, 4-warp CTAs: the smallest grids
        switch (ly) {
            case 8: return launch_sf3x3<8, 1, 4>(map, p, st);
            case 4: return launch_sf3x3<4, 1, 4>(map, p, st);
            case 2: return launch_sf3x3<2, 1, 4>(map, p, st);
            default: break;
        }
    }
    switch (ly * 16 + kt) {
        case 8 * 16 + 4: return launch_sf3x3<8, 4>(map, p, st);
        case 4 * 16 + 4: return launch_sf3x3<4, 4>(map, p, st);
        case 2 * 16 + 4: return launch_sf3x3<2, 4>(map, p, st);
        case 8 * 16 + 8: return launch_sf3x3<8, 8>(map, p, st);
        case 4 * 16 + 8: return launch_sf3x3<4, 8>(map, p, st);
        case 2 * 16 + 8: return launch_sf3x3<2, 8>(map, p, st);
        case 8 * 16 + 2: return launch_sf3x3<8, 2>(map, p, st);
        case 4 * 16 + 2: return launch_sf3x3<4, 2>(map, p, st);
        case 2 * 16 + 2: return launch_sf3x3<2, 2>(map, p, st);
        default: set_error("unsupported sub-region height %d / kt %d", ly, kt); return FSCNN_ERR_ARG;
    }
}

}  // extern "C"
