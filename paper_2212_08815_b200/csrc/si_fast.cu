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
// order is free, so each weight is loaded once per (warp, channel) into registers and
// reused for every nonzero input of that channel in the warp's output tile.
//
// K >= 64 (two passes, si_tile_lists_kernel then si3x3_tl_kernel):
//   1. tile streams: one warp per output tile merges its input region's node fibers (the
//      reference's per-position channel lists) into ONE stream per tile: for every
//      channel with a nonzero in the region (ascending), its entries {region position,
//      value} in ascending position, closed by a link {NP, next channel}.  Count pass +
//      warp scan + placement pass over the fibers; slots handed out by one atomic per
//      tile (placement varies run to run, contents do not).
//   2. conv: a warp owns one tile and 32*KT filters: KT = 2 (4 x 8 tiles, K < 128) or 4
//      (4 x 4 tiles): the accumulator of an output is KT/2 register pairs (f, f') and
//      every FMA an FFMA2 with the input value broadcast.  Its CTA's warps own
//      consecutive tiles of the same filters, so the per-channel weight lines they load
//      (9 x KT x 128 bytes) are mostly L1 hits.  The warp streams its tile's entries
//      through a two-page shared ring with cp.async one page ahead and walks them with
//      one jump-table branch per entry into a block of <= 9 x KT/2 FFMA2 with
//      compile-time registers (si3x3_cases.inc).  No CTA barriers: warps are
//      independent.  Measured bound (ncu, VGG16 layer 8, 90 % input zeros): the
//      indirect branch rate (~1 per 14-18 cycles per SM whatever the tile shape or
//      occupancy: 4x4/4x6/4x8 tiles at 16-32 warps/SM all ran within 10 %) and the
//      weight stream (L1 60 % busy, 57 % hit); FMAs per branch is the lever (KT 2 -> 4:
//      -20 % time).
// K < 64 keeps the single-pass kernel below (one filter per lane, the region decoded per
// 32-channel chunk in shared memory by the CTA).
// No global atomics on the arithmetic; the summation order per output is fixed
// (channels ascending, then region positions ascending), so results are deterministic
// and independent of the batch, the tile placement and the stream layout.
#include <algorithm>
#include <stdlib.h>

#include "common.cuh"

namespace fscnn {
namespace {

#include "si3x3_cases.inc"

constexpr int kSiCC = 32;  // channels per shared-memory chunk

template <int KT> struct SiAcc;
template <> struct SiAcc<1> { using T = float; };

// K < 64: one filter per lane (lane l of warp w owns filter w*32 + l).
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
            si_chan<TY, TX>(acc, wc, ents_base + 8u * (uint32_t)ch_off[c]);
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

// Bank geometry for a layer of K filters: KT filters per lane and Kp = K padded with
// zero filters.  K >= 64: two filters per lane in 64-filter warp groups (the two-pass
// kernel); K < 64: one filter per lane, NW = 2 warps of the single-pass kernel.
struct SiGeom {
    int kt, nw, kp;
};
inline SiGeom si_fast_geom(int k) {
    SiGeom g;
    if (k >= 64) {
        g.kt = k >= 128 ? 4 : 2, g.nw = 0;
        g.kp = (int)ceil_div(k, 32 * g.kt) * 32 * g.kt;
    } else {
        g.kt = 1, g.nw = 2;
        g.kp = 64;
    }
    return g;
}

// ---- K >= 64: tile streams + conv --------------------------------------------------

constexpr int kPg = 256;  // entries per stream page (2 KB): the conv kernel's cp.async unit
constexpr int kOvf = 64;  // ring overflow: a mirror of the head of the page in slot 0

// Output tile TY x TX of one warp; its input region (TY + 2) x (TX + 2) has NP <= 64
// positions; a channel block is <= NP entries + its link.
template <int TY, int TX> struct SiTile {
    static constexpr int RX = TX + 2, NP = (TY + 2) * RX, NA = TY * TX;
    static_assert(NP < kOvf && TY % 2 == 0 && TX % 2 == 0, "tile");
};

// Pass 1: one warp per (tile, image), SI_LW tiles per CTA, no CTA barriers.  Stream =
// head link {NP, first channel}, then per live channel (ascending) its entries {pos,
// value} (positions ascending) and a link {NP, next channel or -1}.  Channels go in
// blocks of SI_CB: pass A reads every region fiber (32-node coalesced windows, lane =
// node) and counts nodes per channel (shared atomics: a fiber's channels are distinct);
// a warp scan places the channel blocks; pass B re-reads the fibers in the same order
// and writes each node at its block start + its rank (positions are visited in
// ascending order, so the rank order is the position order).  Slots are handed out by
// one atomic per tile (placement varies run to run, contents do not).
constexpr int SI_LW = 4, SI_CB = 512;
template <int TY, int TX>
__global__ void __launch_bounds__(SI_LW * 32) si_tile_lists_kernel(
    const int2 *__restrict__ nodes, const int64_t *__restrict__ seg_off, int64_t n_nodes, int n, int c_n, int h,
    int w, int tiles_x, int tpi, unsigned long long *__restrict__ slot_ctr, int64_t cap_slots,
    int64_t *__restrict__ tile_start, int2 *__restrict__ slots) {
    constexpr int kNP = SiTile<TY, TX>::NP, kRX = SiTile<TY, TX>::RX;
    __shared__ int cnt_s[SI_LW][SI_CB], st_s[SI_LW][SI_CB];
    __shared__ int64_t qa_s[SI_LW][kNP], qe_s[SI_LW][kNP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * SI_LW + warp, img = blockIdx.y;
    if (tile >= tpi) return;
    int(&cnt)[SI_CB] = cnt_s[warp];
    int(&st)[SI_CB] = st_s[warp];
    int64_t(&qa)[kNP] = qa_s[warp];
    int64_t(&qe)[kNP] = qe_s[warp];
    const int ty0 = (tile / tiles_x) * TY, tx0 = (tile % tiles_x) * TX;
    const int64_t nseg = (int64_t)n * w * h;
    int64_t nnz = 0;
    for (int p = lane; p < kNP; p += 32) {
        const int yy = ty0 - 1 + p / kRX, xx = tx0 - 1 + p % kRX;
        int64_t q = 0, e = 0;
        if (yy >= 0 && yy < h && xx >= 0 && xx < w) {
            const int64_t i = ((int64_t)img * w + xx) * h + yy;
            q = seg_off[i];
            e = (i + 1 < nseg ? seg_off[i + 1] : n_nodes) - 1;  // the fiber's sentinel
        }
        qa[p] = q, qe[p] = e;
        nnz += e - q;
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) nnz += __shfl_xor_sync(0xffffffffu, nnz, d);
    int64_t base = 0;
    if (lane == 0) {
        // entries + one link per live channel + the head link
        const int64_t need = nnz + (nnz < c_n ? nnz : (int64_t)c_n) + 1;
        base = (int64_t)atomicAdd(slot_ctr, (unsigned long long)need);
        if (base + need > cap_slots) base = -1;  // cannot happen: cap_slots bounds the sum
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    tile_start[(int64_t)img * tpi + tile] = base;
    if (base < 0) return;
    int64_t out = base + 1;  // next free slot
    int64_t link = base;     // the slot waiting for the next live channel
    for (int cb0 = 0; cb0 < c_n; cb0 += SI_CB) {
        const int cbn = min(SI_CB, c_n - cb0);
        for (int i = lane; i < cbn; i += 32) cnt[i] = 0;
        __syncwarp();
        // pass A: count per channel
        for (int p = 0; p < kNP; ++p) {
            const int64_t e = qe[p];
            for (int64_t q = qa[p]; q < e; q += 32) {
                const int c = q + lane < e ? __ldg(&nodes[q + lane].x) - cb0 : SI_CB;
                if (c < cbn) atomicAdd(&cnt[c], 1);
                if (__any_sync(0xffffffffu, c >= cbn && q + lane < e)) break;  // rest in later blocks
            }
        }
        __syncwarp();
        // place the blocks: lane-strided groups of 32 channels, running offset
        int64_t boff = 0;
        for (int g0 = 0; g0 < cbn; g0 += 32) {
            const int ci = g0 + lane;
            const int k = ci < cbn ? cnt[ci] : 0;
            const int size = k ? k + 1 : 0;
            int inc = size;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int o = __shfl_up_sync(0xffffffffu, inc, d);
                if (lane >= d) inc += o;
            }
            const unsigned live = __ballot_sync(0xffffffffu, k > 0);
            const int64_t start = out + boff + inc - size;
            if (ci < cbn) st[ci] = (int)(boff + inc - size);
            if (live) {
                const int first = __ffs(live) - 1;
                if (lane == 0) slots[link] = make_int2(kNP, cb0 + g0 + first);
                const unsigned after = lane < 31 ? live & (0xfffffffeu << lane) : 0u;
                if (k && after) slots[start + k] = make_int2(kNP, cb0 + g0 + __ffs(after) - 1);
                link = __shfl_sync(0xffffffffu, start + k, 31 - __clz(live));
            }
            boff += __shfl_sync(0xffffffffu, inc, 31);
        }
        for (int i = lane; i < cbn; i += 32) cnt[i] = 0;
        __syncwarp();
        // pass B: the same walk, every node to its block start + rank
        for (int p = 0; p < kNP; ++p) {
            const int64_t e = qe[p];
            int64_t q = qa[p];
            for (; q < e; q += 32) {
                int2 nd = make_int2(SI_CB + cb0, 0);
                if (q + lane < e) nd = __ldg(&nodes[q + lane]);
                const int c = nd.x - cb0;
                if (c < cbn) {
                    const int rk = atomicAdd(&cnt[c], 1);
                    slots[out + st[c] + rk] = make_int2(p, nd.y);
                }
                const unsigned beyond = __ballot_sync(0xffffffffu, c >= cbn && q + lane < e);
                if (beyond) {  // the fiber continues in a later channel block
                    q += __ffs(beyond) - 1;
                    break;
                }
            }
            if (lane == 0) qa[p] = q < e ? q : e;
        }
        out += boff;
        __syncwarp();
    }
    if (lane == 0) slots[link] = make_int2(kNP, -1);
}

// Pass 1 from a dense NCHW activation instead of nodes (the batched network forward: no
// encode between layers).  The same stream, entry for entry: per live channel ascending,
// the region positions whose value is stored by the reference encoder (value != +-0.0;
// NaN kept -- sparsify_tensor3, sparse_core.py:334-353) in ascending position order, the
// same links.  Lanes own region positions (a row of the window is contiguous); a count
// pass sizes the tile's stream, a second pass writes it channel by channel (the dense
// input gives each channel's entries and their ranks with one ballot, no shared memory).
template <int TY, int TX>
__global__ void __launch_bounds__(SI_LW * 32) si_tile_lists_dense_kernel(
    const float *__restrict__ x, int c_n, int h, int w, int tiles_x, int tpi,
    unsigned long long *__restrict__ slot_ctr, int64_t cap_slots, int64_t *__restrict__ tile_start,
    int2 *__restrict__ slots) {
    constexpr int kNP = SiTile<TY, TX>::NP, kRX = SiTile<TY, TX>::RX;
    constexpr int kR = (kNP + 31) / 32;  // lane rounds over the region positions
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int tile = blockIdx.x * SI_LW + warp, img = blockIdx.y;
    if (tile >= tpi) return;
    const int ty0 = (tile / tiles_x) * TY, tx0 = (tile % tiles_x) * TX;
    int64_t off[kR];  // this lane's position in a channel plane, or -1 outside the image
#pragma unroll
    for (int r = 0; r < kR; ++r) {
        const int p = r * 32 + lane;
        const int yy = ty0 - 1 + p / kRX, xx = tx0 - 1 + p % kRX;
        off[r] = (p < kNP && yy >= 0 && yy < h && xx >= 0 && xx < w) ? (int64_t)yy * w + xx : -1;
    }
    const float *xi = x + (int64_t)img * c_n * h * w;
    const int64_t plane = (int64_t)h * w;
    auto stored = [&](int ch, int r) -> bool {
        if (off[r] < 0) return false;
        return (__float_as_uint(__ldg(xi + ch * plane + off[r])) & 0x7fffffffu) != 0u;
    };
    int64_t nnz = 0, live = 0;
    for (int ch = 0; ch < c_n; ++ch) {
        int k = 0;
#pragma unroll
        for (int r = 0; r < kR; ++r) k += __popc(__ballot_sync(0xffffffffu, stored(ch, r)));
        nnz += k;
        live += k > 0;
    }
    int64_t base = 0;
    if (lane == 0) {
        const int64_t need = nnz + live + 1;
        base = (int64_t)atomicAdd(slot_ctr, (unsigned long long)need);
        if (base + need > cap_slots) base = -1;  // cannot happen: cap_slots bounds the sum
    }
    base = __shfl_sync(0xffffffffu, base, 0);
    tile_start[(int64_t)img * tpi + tile] = base;
    if (base < 0) return;
    int64_t link = base, out = base + 1;
    for (int ch = 0; ch < c_n; ++ch) {
        unsigned m[kR];
        float v[kR];
        int k = 0;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            v[r] = off[r] >= 0 ? __ldg(xi + ch * plane + off[r]) : 0.0f;
            m[r] = __ballot_sync(0xffffffffu, off[r] >= 0 && (__float_as_uint(v[r]) & 0x7fffffffu) != 0u);
            k += __popc(m[r]);
        }
        if (!k) continue;
        if (lane == 0) slots[link] = make_int2(kNP, ch);
        int before = 0;
#pragma unroll
        for (int r = 0; r < kR; ++r) {
            if ((m[r] >> lane) & 1u)
                slots[out + before + __popc(m[r] & ((1u << lane) - 1u))] = make_int2(r * 32 + lane, __float_as_int(v[r]));
            before += __popc(m[r]);
        }
        link = out + k;
        out += k + 1;
    }
    if (lane == 0) slots[link] = make_int2(kNP, -1);
}

// Epilogue of the two-pass kernel: + bias (and Alg. 7's fused 2x2 pool, layers.py:345-390,
// in pool2d's order -- (ph, pw) row-major, max from -inf with '>', avg as a left-to-right
// sum (first NaN wins) / 4 -- before the bias), a zero sum stored as +0.0 (no node in
// the reference).  Lane owns filters grp*64 + lane (low half) and grp*64 + 32 + lane.
template <int kTY, int kTX, int PAIRS>
__device__ __forceinline__ void si_store_pairs(const unsigned long long (&acc)[kTY * kTX * PAIRS], int grp, int lane,
                                               int img, int ty0, int tx0, int h, int w, int k_n,
                                               const float *__restrict__ bias, float *__restrict__ y, int pool) {
#pragma unroll
    for (int j = 0; j < 2 * PAIRS; ++j) {
        const int k = (grp * 2 * PAIRS + j) * 32 + lane;
        if (k >= k_n) continue;
        const float bk = bias ? bias[k] : 0.0f;
        if (pool) {
            const int ho = h >> 1, wo = w >> 1;
            float *yk = y + ((int64_t)img * k_n + k) * ho * wo;
#pragma unroll
            for (int qy = 0; qy < kTY / 2; ++qy) {
                const int yy = (ty0 >> 1) + qy;
                if (yy >= ho) break;
#pragma unroll
                for (int qx = 0; qx < kTX / 2; ++qx) {
                    const int xx = (tx0 >> 1) + qx;
                    if (xx >= wo) break;
                    float m = pool == 1 ? -INFINITY : 0.0f;
#pragma unroll
                    for (int ph = 0; ph < 2; ++ph)
#pragma unroll
                        for (int pw = 0; pw < 2; ++pw) {
                            const int o = (2 * qy + ph) * kTX + 2 * qx + pw;
                            float v = __uint_as_float((unsigned)(acc[o * PAIRS + (j >> 1)] >> (32 * (j & 1))));
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
        } else {
            float *yk = y + ((int64_t)img * k_n + k) * h * w;
#pragma unroll
            for (int oy = 0; oy < kTY; ++oy) {
                const int yy = ty0 + oy;
                if (yy >= h) break;
#pragma unroll
                for (int ox = 0; ox < kTX; ++ox) {
                    const int xx = tx0 + ox;
                    if (xx >= w) break;
                    float v = __uint_as_float((unsigned)(acc[(oy * kTX + ox) * PAIRS + (j >> 1)] >> (32 * (j & 1))));
                    v = (v != 0.0f) ? v : 0.0f;
                    if (bias) v = __fadd_rn(v, bk);
                    yk[(int64_t)yy * w + xx] = v;
                }
            }
        }
    }
}

// Pass 2: NW warps per CTA, warp = (tile blockIdx.x*NW + warp, filter group blockIdx.y of
// 64*PAIRS filters).  The tile's stream goes through a per-warp shared ring of two 2 KB
// pages (absolute page q of the slot buffer in ring slot q & 1) plus an overflow area
// that mirrors the head of the page in slot 0, so a channel block that runs off the end
// of slot 1 reads on linearly; cp.async keeps the next page in flight, and before a block
// that may reach the next page the warp waits for it.
template <int TY, int TX, int PAIRS, int NW, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    si3x3_tl_kernel(const int2 *__restrict__ slots, const int64_t *__restrict__ tile_start, int n_tiles,
                    int tiles_x, int tiles_per_img, int h, int w, const unsigned long long *__restrict__ wf,
                    int k_n, int kp, const float *__restrict__ bias, float *__restrict__ y, int pool) {
    constexpr int kTY = TY, kTX = TX, kNP = SiTile<TY, TX>::NP;
    __shared__ __align__(16) int2 ring[NW][2 * kPg + kOvf];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int t = blockIdx.x * NW + warp;
    if (t >= n_tiles) return;  // no CTA barriers below: warps are independent
    const int grp = blockIdx.y;
    const int img = t / tiles_per_img, r = t % tiles_per_img;
    const int ty0 = (r / tiles_x) * kTY, tx0 = (r % tiles_x) * kTX;
    unsigned long long acc[kTY * kTX * PAIRS];
#pragma unroll
    for (int i = 0; i < kTY * kTX * PAIRS; ++i) acc[i] = 0ull;
    const int64_t s0 = tile_start[t];
    if (s0 >= 0) {
        const uint32_t ring0 = (uint32_t)__cvta_generic_to_shared(&ring[warp][0]);
        // page q -> ring slot q & 1 (16 bytes per lane per copy); an even page's first
        // kOvf entries also go to the overflow area behind slot 1
        auto fetch = [&](int64_t q) {
            const uint32_t dst = ring0 + (uint32_t)(q & 1) * (kPg * 8) + lane * 16;
            const char *src = reinterpret_cast<const char *>(slots + q * kPg) + lane * 16;
#pragma unroll
            for (int i = 0; i < kPg * 8 / 512; ++i)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + i * 512), "l"(src + i * 512)
                             : "memory");
            if (!(q & 1))
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring0 + 2 * kPg * 8 + lane * 16),
                             "l"(src)
                             : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        };
        int64_t pg = s0 / kPg;  // page of the cursor; pages pg and pg + 1 are issued
        fetch(pg);
        fetch(pg + 1);  // the buffer has a spare page past the last slot handed out
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        __syncwarp();
        bool next_ready = true;  // page pg + 1 has landed
        int64_t pos = s0;        // absolute slot of the cursor
        uint32_t cur = ring0 + (uint32_t)(pos & (2 * kPg - 1)) * 8;
        int lx, ly;
        asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(lx), "=r"(ly) : "r"(cur) : "memory");
        ++pos;
        // bank [C][Kp/(64 PAIRS)][9][32] of PAIRS (f, f') pairs
        const unsigned long long *wk = wf + ((int64_t)grp * 288 + lane) * PAIRS;
        const int64_t ch_stride = (int64_t)(kp / (64 * PAIRS)) * 288 * PAIRS;
        while (ly >= 0) {
            if (pos / kPg != pg) {  // the cursor entered the next page: refill the slot it left
                ++pg;
                if (!next_ready) {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                    __syncwarp();
                }
                fetch(pg + 1);
                next_ready = false;
            }
            if (!next_ready && (pos + kNP) / kPg != pg) {  // this block may reach page pg + 1
                asm volatile("cp.async.wait_group 0;" ::: "memory");
                __syncwarp();
                next_ready = true;
            }
            cur = ring0 + (uint32_t)(pos & (2 * kPg - 1)) * 8;
            unsigned long long wc[9 * PAIRS];
            const unsigned long long *src = wk + ly * ch_stride;
            if constexpr (PAIRS == 2) {
#pragma unroll
                for (int i = 0; i < 9; ++i) {
                    const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2 *>(src + i * 64));
                    wc[2 * i] = v.x, wc[2 * i + 1] = v.y;
                }
            } else {
#pragma unroll
                for (int i = 0; i < 9; ++i) wc[i] = __ldg(src + i * 32);
            }
            const uint32_t c_in = cur;
            si_chanp<kTY, kTX, PAIRS>(acc, wc, cur, lx, ly);
            pos += (cur - c_in) >> 3;
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    si_store_pairs<TY, TX, PAIRS>(acc, grp, lane, img, ty0, tx0, h, w, k_n, bias, y, pool);
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

// Workspace of the two-pass path: [slot counter][tile_start: n_tiles][pad][slots].  The
// slot budget bounds sum over tiles of (region nnz + live channels + 1): every node lies
// in <= 4 tile regions ((TY+2) x (TX+2) regions over TY x TX tiles), every tile has <= C
// live channels; two spare pages cover the conv kernel's read-ahead.
struct SiWs {
    int64_t n_tiles, cap_slots, off_ts, off_slots, bytes;
};
template <int TY, int TX>
inline SiWs si_ws(int n, int c, int h, int w, int64_t n_nodes) {
    SiWs s;
    s.n_tiles = (int64_t)n * ceil_div(w, TX) * ceil_div(h, TY);
    const int64_t inreg = 4 * n_nodes;
    s.cap_slots = inreg + std::min<int64_t>(s.n_tiles * c, inreg) + s.n_tiles;
    s.off_ts = 256;
    s.off_slots = (s.off_ts + 8 * s.n_tiles + 255) / 256 * 256;
    s.bytes = s.off_slots + (ceil_div(s.cap_slots, kPg) + 2) * (int64_t)kPg * 8;
    return s;
}

template <int TY, int TX, int PAIRS, int NW, int MINB>
int launch_tl(const int2 *nodes, const int64_t *seg_off, int64_t n_nodes, int n, int c, int h, int w,
              const float *wf, int k, int kp, const float *bias, float *y, cudaStream_t st, int pool,
              const float *x_dense = nullptr) {
    // dense input: the node-count bound is the element count
    const SiWs s = si_ws<TY, TX>(n, c, h, w, x_dense ? (int64_t)n * c * h * w : n_nodes);
    static bool pool_set = false;
    if (!pool_set) {
        // keep freed workspace in the stream-ordered pool (no OS round trip per call)
        int dev = 0;
        cudaMemPool_t mp;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&mp, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool_set = true;
    }
    char *ws = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void **>(&ws), (size_t)s.bytes, st) != cudaSuccess) {
        cudaGetLastError();
        set_error("si3x3 fast: workspace of %lld bytes could not be allocated", (long long)s.bytes);
        return FSCNN_ERR_CUDA;
    }
    cudaMemsetAsync(ws, 0, 8, st);
    const int tiles_x = (int)ceil_div(w, TX), tpi = tiles_x * (int)ceil_div(h, TY);
    auto *ctr = reinterpret_cast<unsigned long long *>(ws);
    auto *ts = reinterpret_cast<int64_t *>(ws + s.off_ts);
    auto *slots = reinterpret_cast<int2 *>(ws + s.off_slots);
    int rc;
    if (x_dense) {
        si_tile_lists_dense_kernel<TY, TX><<<dim3((unsigned)ceil_div(tpi, SI_LW), (unsigned)n), SI_LW * 32, 0, st>>>(
            x_dense, c, h, w, tiles_x, tpi, ctr, s.cap_slots, ts, slots);
        rc = check_launch("si_tile_lists_dense_kernel");
    } else {
        si_tile_lists_kernel<TY, TX><<<dim3((unsigned)ceil_div(tpi, SI_LW), (unsigned)n), SI_LW * 32, 0, st>>>(
            nodes, seg_off, n_nodes, n, c, h, w, tiles_x, tpi, ctr, s.cap_slots, ts, slots);
        rc = check_launch("si_tile_lists_kernel");
    }
    if (rc == FSCNN_OK) {
        dim3 grid((unsigned)ceil_div(s.n_tiles, NW), (unsigned)(kp / (64 * PAIRS)));
        si3x3_tl_kernel<TY, TX, PAIRS, NW, MINB><<<grid, NW * 32, 0, st>>>(
            slots, ts, (int)s.n_tiles, tiles_x, tpi, h, w, reinterpret_cast<const unsigned long long *>(wf), k,
            kp, bias, y, pool);
        rc = check_launch("si3x3_tl_kernel");
    }
    cudaFreeAsync(ws, st);
    return rc;
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
    const int2 *nd = reinterpret_cast<const int2 *>(in_nodes);
    cudaStream_t st = as_stream(stream);
    if (g.kt >= 2) {
        FSCNN_REQUIRE(n * (int64_t)ceil_div(w, 4) * ceil_div(h, 4) < (1ll << 31), "too many tiles");
        // 4 filters per lane on 4 x 4 tiles from K = 128 (twice the FMAs per jump-table
        // branch of 2 filters on 4 x 8, the better trade once K fills 128-filter groups)
        if (g.kt == 2) return launch_tl<4, 8, 1, 4, 5>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, g.kp, bias, y, st, pool);
        return launch_tl<4, 4, 2, 4, 4>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, g.kp, bias, y, st, pool);
    }
    // one filter per lane (K < 64)
    return launch_fast<4, 8, 2, 1>(nd, in_seg_off, n_nodes, n, c, h, w, wf, k, g.kp, bias, y, st, pool);
}

int fscnn_si_conv3x3_fast_dense(const float *x, int n, int c, int h, int w, const float *wf, int k,
                                const float *bias, int pool, float *y, void *stream) {
    FSCNN_REQUIRE(pool >= 0 && pool <= 2, "pool must be 0 (none), 1 (2x2 max) or 2 (2x2 avg)");
    if (pool) FSCNN_REQUIRE(h % 2 == 0 && w % 2 == 0, "fused 2x2 pool needs even extents");
    FSCNN_REQUIRE(n >= 0 && c > 0 && h > 0 && w > 0 && k >= 0, "bad extents");
    if (n == 0 || k == 0) return FSCNN_OK;
    FSCNN_REQUIRE(x && wf && y, "null buffer");
    FSCNN_REQUIRE(n <= 65535, "batch too large for one launch (%d > 65535)", n);
    const SiGeom g = si_fast_geom(k);
    FSCNN_REQUIRE(g.kt >= 2, "the dense-input path needs K >= 64 (got %d)", k);
    FSCNN_REQUIRE(n * (int64_t)ceil_div(w, 4) * ceil_div(h, 4) < (1ll << 31), "too many tiles");
    cudaStream_t st = as_stream(stream);
    if (g.kt == 2)
        return launch_tl<4, 8, 1, 4, 5>(nullptr, nullptr, 0, n, c, h, w, wf, k, g.kp, bias, y, st, pool, x);
    return launch_tl<4, 4, 2, 4, 4>(nullptr, nullptr, 0, n, c, h, w, wf, k, g.kp, bias, y, st, pool, x);
}

int fscnn_si_conv3x3_fast(const fscnn_node *in_nodes, const int64_t *in_seg_off, int64_t n_nodes, int n,
                          int c, int h, int w, const float *wf, int k, const float *bias, float *y,
                          void *stream) {
    return fscnn_si_conv3x3_fast_pool(in_nodes, in_seg_off, n_nodes, n, c, h, w, wf, k, bias, 0, y, stream);
}

}  // extern "C"
