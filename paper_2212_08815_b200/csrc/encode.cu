// Dense <-> node-format conversion on the device, bit-exact with the reference
// encoder (sparse_core.py:319-353, SparseTensor4.stack :273-290) and decoder
// (densify_tensor3, sparse_core.py:356-368).
//
// Encoding is count -> exclusive scan of (count + 1) -> ordered write, exactly the
// reference's bincount/cumsum/scatter, so offsets and node order match by
// construction.  Two source walkers:
//   * thread-per-segment: one thread scans one inner fiber (any stride); used when
//     the inner axis is strided (e.g. CHW nodes from NCHW activations -- adjacent
//     threads then read adjacent addresses of the mid axis... or stride-W rows);
//   * warp-per-segment: a warp scans a contiguous fiber 32 values at a time and
//     compacts with ballot/popc, preserving order;
//   * tiled (write pass only, strided inner over a unit-stride outer axis): a CTA
//     stages a 32 x 8 position x 32 channel tile in shared memory and warps then
//     compact segment by segment as in the warp walker (write_tile_kernel).
// The scan is a three-kernel block scan over int64 (4096 segments per block).
#include "common.cuh"

namespace fscnn {
namespace {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 4;
constexpr int kScanTile = kScanThreads * kScanItems;

// --- source walkers ----------------------------------------------------------

// Thread t -> segment id for the thread-per-segment kernels.  Segments are numbered
// (b, o, m) with m fastest; when the outer axis has the smaller memory stride (e.g. CHW
// nodes of NCHW activations: segment (w, h), channels strided) neighbouring threads
// take neighbouring o instead, so their fiber reads coalesce.
__device__ __forceinline__ int64_t seg_of_thread(int64_t t, int64_t outer, int64_t mid, bool o_fast) {
    if (!o_fast) return t;
    const int64_t per = outer * mid;
    const int64_t b = t / per, r = t - b * per;
    const int64_t m = r / outer, o = r - m * outer;
    return (b * outer + o) * mid + m;
}

struct StridedSrc {
    const float *p;
    int64_t outer, mid, inner, s_b, s_o, s_m, s_i;
    bool o_fast;
    __device__ __forceinline__ int64_t seg(int64_t t) const { return seg_of_thread(t, outer, mid, o_fast); }
    struct Fiber {
        const float *p;
    };
    __device__ __forceinline__ Fiber fiber(int64_t s) const {
        int64_t m = s % mid;
        int64_t bo = s / mid;
        int64_t o = bo % outer;
        int64_t b = bo / outer;
        return {p + b * s_b + o * s_o + m * s_m};
    }
    __device__ __forceinline__ float at(Fiber f, int64_t i) const { return f.p[i * s_i]; }
    __device__ __forceinline__ bool present(Fiber f, int64_t i) const { return at(f, i) != 0.0f; }
};

// A strided value view plus a presence mask with the same element offsets: an entry is
// stored iff its mask byte is set, whatever its value (node-preserving transposes keep
// explicit zero-valued nodes this way).
struct MaskedSrc {
    const float *p;
    const uint8_t *m;
    int64_t outer, mid, inner, s_b, s_o, s_m, s_i;
    bool o_fast;
    __device__ __forceinline__ int64_t seg(int64_t t) const { return seg_of_thread(t, outer, mid, o_fast); }
    struct Fiber {
        const float *p;
        const uint8_t *m;
    };
    __device__ __forceinline__ Fiber fiber(int64_t s) const {
        int64_t mm = s % mid;
        int64_t bo = s / mid;
        int64_t off = (bo / outer) * s_b + (bo % outer) * s_o + mm * s_m;
        return {p + off, m + off};
    }
    __device__ __forceinline__ float at(Fiber f, int64_t i) const { return f.p[i * s_i]; }
    __device__ __forceinline__ bool present(Fiber f, int64_t i) const { return f.m[i * s_i] != 0; }
};

// Fast-path filter packing: segment s = g*C + c; inner i = kl*9 + tap reads
// W[g*kt + kl][c][tap] from a dense [K][C][3][3] bank (zero past K).
struct SfPackSrc {
    const float *w;
    int64_t k, c, kt;
    int64_t inner;
    __device__ __forceinline__ int64_t seg(int64_t t) const { return t; }
    struct Fiber {
        const float *p;
        int64_t kmax;
    };
    __device__ __forceinline__ Fiber fiber(int64_t s) const {
        int64_t g = s / c, ch = s % c;
        int64_t kmax = k - g * kt;
        return {w + ((g * kt) * c + ch) * 9, kmax < kt ? kmax : kt};
    }
    __device__ __forceinline__ float at(Fiber f, int64_t i) const {
        int64_t kl = i / 9, tap = i - kl * 9;
        return kl < f.kmax ? f.p[kl * c * 9 + tap] : 0.0f;
    }
    __device__ __forceinline__ bool present(Fiber f, int64_t i) const { return at(f, i) != 0.0f; }
};

template <class Src>
__global__ void count_thread_kernel(Src src, int64_t n_seg, int64_t *cnt) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_seg) return;
    const int64_t s = src.seg(t);
    auto b = src.fiber(s);
    int64_t n = 0;
#pragma unroll 8
    for (int64_t i = 0; i < src.inner; ++i) n += src.present(b, i);
    cnt[s] = n + 1;
}

template <class Src>
__global__ void count_warp_kernel(Src src, int64_t n_seg, int64_t *cnt) {
    int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (s >= n_seg) return;
    auto b = src.fiber(s);
    int64_t n = 0;
    for (int64_t i0 = 0; i0 < src.inner; i0 += 32) {
        int64_t i = i0 + lane;
        bool nz = (i < src.inner) && src.present(b, i);
        n += __popc(__ballot_sync(0xffffffffu, nz));
    }
    if (lane == 0) cnt[s] = n + 1;
}

template <class Src>
__global__ void write_thread_kernel(Src src, int64_t n_seg, const int64_t *seg_off, int2 *nodes,
                                    int sentinel) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_seg) return;
    const int64_t s = src.seg(t);
    auto b = src.fiber(s);
    int64_t p = seg_off[s];
#pragma unroll 8
    for (int64_t i = 0; i < src.inner; ++i)
        if (src.present(b, i)) nodes[p++] = make_int2((int)i, __float_as_int(src.at(b, i)));
    nodes[p] = make_int2(sentinel, 0);
}

template <class Src>
__global__ void write_warp_kernel(Src src, int64_t n_seg, const int64_t *seg_off, int2 *nodes,
                                  int sentinel) {
    int64_t s = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (s >= n_seg) return;
    auto b = src.fiber(s);
    int64_t p = seg_off[s];
    const unsigned lt = (1u << lane) - 1u;
    for (int64_t i0 = 0; i0 < src.inner; i0 += 32) {
        int64_t i = i0 + lane;
        bool nz = (i < src.inner) && src.present(b, i);
        float v = nz ? src.at(b, i) : 0.0f;
        unsigned m = __ballot_sync(0xffffffffu, nz);
        if (nz) nodes[p + __popc(m & lt)] = make_int2((int)i, __float_as_int(v));
        p += __popc(m);
    }
    if (lane == 0) nodes[p] = make_int2(sentinel, 0);
}

// Tiled writer for a strided inner axis over a unit-stride outer axis (CHW nodes of NCHW
// activations: segment (w, h), channels H*W apart).  The per-thread walker above reads
// coalesced but every thread appends to its own node run, so each store instruction
// touches 32 scattered 8-byte slots (partial-sector writes: measured 130 MB written and
// 180 MB read for a 103 MB input and 106 MB of nodes).  Here a CTA owns a tile of kTO outer x kTM mid
// positions: per 32-channel chunk it stages the tile in shared memory with rows along
// the unit-stride axis (coalesced loads), then each warp walks its 32 segments one at a
// time, lanes over channels, ballot-compacting into the segment's run (coalesced stores,
// node order unchanged).  The warp's running write positions live one per lane.
constexpr int kTO = 32, kTM = 8, kTC = 32, kTilePitch = kTO * kTM + 1;

__global__ void __launch_bounds__(256) write_tile_kernel(StridedSrc src, int64_t n_otile,
                                                         int64_t n_mtile, const int64_t *seg_off,
                                                         int2 *nodes, int sentinel) {
    __shared__ float tile[kTC * kTilePitch];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    int64_t bid = blockIdx.x;
    const int64_t ot = bid % n_otile;
    bid /= n_otile;
    const int64_t mt = bid % n_mtile, b = bid / n_mtile;
    const int64_t o0 = ot * kTO, m0 = mt * kTM;
    // lane j of warp w owns segment (o0 + 4w + j/8, m0 + j%8): for a fixed o its 8 mids
    // are consecutive segment ids.
    const int my_o = wid * 4 + (lane >> 3), my_m = lane & 7;
    const bool my_ok = o0 + my_o < src.outer && m0 + my_m < src.mid;
    int64_t pl = my_ok ? seg_off[(b * src.outer + o0 + my_o) * src.mid + m0 + my_m] : 0;
    const unsigned valid_lanes = __ballot_sync(0xffffffffu, my_ok);
    const unsigned lt = (1u << lane) - 1u;
    const float *base = src.p + b * src.s_b + o0 + m0 * src.s_m;
    const bool ld_o = o0 + lane < src.outer;
    for (int64_t c0 = 0; c0 < src.inner; c0 += kTC) {
        __syncthreads();
#pragma unroll 8
        for (int r = wid; r < kTC * kTM; r += 8) {   // row r = (channel, mid) pair
            const int ch = r / kTM, m = r % kTM;
            float v = 0.0f;
            if (ld_o && c0 + ch < src.inner && m0 + m < src.mid)
                v = __ldg(base + (c0 + ch) * src.s_i + m * src.s_m + lane);
            tile[ch * kTilePitch + m * kTO + lane] = v;
        }
        __syncthreads();
        const bool ch_ok = c0 + lane < src.inner;
        for (int j = 0; j < 32; ++j) {
            if (!((valid_lanes >> j) & 1u)) continue;
            const int o = wid * 4 + (j >> 3), m = j & 7;
            const float v = tile[lane * kTilePitch + m * kTO + o];
            const bool nz = ch_ok && v != 0.0f;
            const unsigned bal = __ballot_sync(0xffffffffu, nz);
            const int64_t p = __shfl_sync(0xffffffffu, pl, j);
            if (nz) nodes[p + __popc(bal & lt)] = make_int2((int)(c0 + lane), __float_as_int(v));
            if (lane == j) pl += __popc(bal);
        }
    }
    if (my_ok) nodes[pl] = make_int2(sentinel, 0);
}

inline bool use_tile_writer(const StridedSrc &s) {
    return s.s_o == 1 && s.s_i != 1 && s.inner >= 16 && s.outer >= 16;
}

// --- int64 exclusive scan -------------------------------------------------------

__device__ __forceinline__ int64_t warp_incl_scan(int64_t v) {
    int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        int64_t t = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += t;
    }
    return v;
}

// Block-wide exclusive scan of one value per thread; returns exclusive prefix, *total = sum.
__device__ int64_t block_excl_scan(int64_t v, int64_t *total) {
    __shared__ int64_t warp_sums[32];
    __shared__ int64_t block_total;
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int64_t incl = warp_incl_scan(v);
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
        int nw = blockDim.x >> 5;
        int64_t w = lane < nw ? warp_sums[lane] : 0;
        int64_t wi = warp_incl_scan(w);
        if (lane < nw) warp_sums[lane] = wi - w;
        if (lane == nw - 1) block_total = wi;
    }
    __syncthreads();
    int64_t excl = warp_sums[wid] + incl - v;
    if (total) *total = block_total;
    __syncthreads();
    return excl;
}

__global__ void scan_tiles_kernel(int64_t *a, int64_t n, int64_t *tile_sums) {
    int64_t base = blockIdx.x * (int64_t)kScanTile + threadIdx.x * (int64_t)kScanItems;
    int64_t v[kScanItems];
    int64_t sum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = (base + j < n) ? a[base + j] : 0;
        sum += v[j];
    }
    int64_t tot;
    int64_t run = block_excl_scan(sum, &tot);
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n) a[base + j] = run;
        run += v[j];
    }
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

// One block scans all tile sums (exclusive, in place); writes the grand total.
__global__ void scan_sums_kernel(int64_t *sums, int64_t n, int64_t *total) {
    int64_t per = (n + blockDim.x - 1) / blockDim.x;
    int64_t lo = threadIdx.x * per, hi = min(n, lo + per);
    int64_t s = 0;
    for (int64_t i = lo; i < hi; ++i) s += sums[i];
    int64_t tot;
    int64_t run = block_excl_scan(s, &tot);
    for (int64_t i = lo; i < hi; ++i) {
        int64_t t = sums[i];
        sums[i] = run;
        run += t;
    }
    if (threadIdx.x == 0) *total = tot;
}

__global__ void scan_add_kernel(int64_t *a, int64_t n, const int64_t *tile_sums) {
    int64_t base = blockIdx.x * (int64_t)kScanTile;
    int64_t add = tile_sums[blockIdx.x];
    if (add == 0) return;
    for (int j = threadIdx.x; j < kScanTile; j += blockDim.x)
        if (base + j < n) a[base + j] += add;
}

__global__ void side_tables_kernel(const int64_t *seg_off, int64_t n_seg, int64_t mid,
                                   int64_t per_tensor, int64_t *matrix_off, int64_t *tensor_off) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    if (matrix_off && s % mid == 0) matrix_off[s / mid] = seg_off[s];
    if (tensor_off && s % per_tensor == 0) tensor_off[s / per_tensor] = seg_off[s];
}

int scan_inplace(int64_t *a, int64_t n, int64_t *total, void *ws, size_t ws_bytes,
                 cudaStream_t st) {
    int64_t tiles = ceil_div(n, kScanTile);
    FSCNN_REQUIRE(ws_bytes >= (size_t)tiles * sizeof(int64_t) && ws != nullptr,
                  "encode workspace too small (%zu bytes, need %lld)", ws_bytes,
                  (long long)(tiles * 8));
    int64_t *sums = static_cast<int64_t *>(ws);
    scan_tiles_kernel<<<(unsigned)tiles, kScanThreads, 0, st>>>(a, n, sums);
    FSCNN_LAUNCH_CHECK("scan_tiles_kernel");
    scan_sums_kernel<<<1, kScanThreads, 0, st>>>(sums, tiles, total);
    FSCNN_LAUNCH_CHECK("scan_sums_kernel");
    if (tiles > 1) {
        scan_add_kernel<<<(unsigned)tiles, 256, 0, st>>>(a, n, sums);
        FSCNN_LAUNCH_CHECK("scan_add_kernel");
    }
    return FSCNN_OK;
}

// Warp-per-segment pays off only when fibers are contiguous and long enough.
inline bool use_warp_walker(int64_t inner, int64_t s_i) { return s_i == 1 && inner >= 32; }

template <class Src>
int encode_offsets_impl(const Src &src, int64_t n_seg, bool warp_mode, int64_t *seg_off,
                        int64_t *total, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (n_seg == 0) {
        cudaMemsetAsync(total, 0, sizeof(int64_t), st);
        return check_launch("memset total");
    }
    if (warp_mode) {
        count_warp_kernel<<<(unsigned)ceil_div(n_seg * 32, 256), 256, 0, st>>>(src, n_seg, seg_off);
        FSCNN_LAUNCH_CHECK("count_warp_kernel");
    } else {
        count_thread_kernel<<<(unsigned)ceil_div(n_seg, 256), 256, 0, st>>>(src, n_seg, seg_off);
        FSCNN_LAUNCH_CHECK("count_thread_kernel");
    }
    return scan_inplace(seg_off, n_seg, total, ws, ws_bytes, st);
}

template <class Src>
int encode_nodes_impl(const Src &src, int64_t n_seg, bool warp_mode, const int64_t *seg_off,
                      fscnn_node *nodes, cudaStream_t st, int sentinel = -1) {
    if (n_seg == 0) return FSCNN_OK;
    int2 *out = reinterpret_cast<int2 *>(nodes);
    if (warp_mode) {
        write_warp_kernel<<<(unsigned)ceil_div(n_seg * 32, 256), 256, 0, st>>>(src, n_seg, seg_off, out, sentinel);
        FSCNN_LAUNCH_CHECK("write_warp_kernel");
    } else {
        write_thread_kernel<<<(unsigned)ceil_div(n_seg, 256), 256, 0, st>>>(src, n_seg, seg_off, out, sentinel);
        FSCNN_LAUNCH_CHECK("write_thread_kernel");
    }
    return FSCNN_OK;
}

// --- decoder ----------------------------------------------------------------------

// mask (optional, same element offsets as dst) receives 1 where a node is stored
__global__ void decode_kernel(const int2 *nodes, const int64_t *seg_off, int64_t n_seg,
                              int64_t outer, int64_t mid, int64_t inner, float *dst, uint8_t *mask,
                              int64_t d_b, int64_t d_o, int64_t d_m, int64_t d_i) {
    int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_seg) return;
    const int64_t s = seg_of_thread(t, outer, mid, d_o < d_m);  // coalesced destination writes
    int64_t m = s % mid, bo = s / mid, o = bo % outer, b = bo / outer;
    const int64_t off = b * d_b + o * d_o + m * d_m;
    float *d = dst + off;
    int64_t p = seg_off[s];
    int2 nd = nodes[p];
    for (int64_t i = 0; i < inner; ++i) {
        float v = 0.0f;
        const bool hit = nd.x == i;
        if (hit) {
            v = __int_as_float(nd.y);
            nd = nodes[++p];
        }
        d[i * d_i] = v;
        if (mask) mask[off + i * d_i] = hit;
    }
}

// --- segment gather ------------------------------------------------------------------
// New segment j is a copy of old segment map[j] (its nodes and sentinel, values and
// indices untouched -- explicit zero-valued nodes survive), or empty (sentinel only)
// when map[j] < 0.  pad_tensor on CHW nodes (layers.py:521-535) is this gather.

__device__ __forceinline__ int64_t old_seg_len(const int64_t *off, int64_t n, int64_t total, int64_t s) {
    return ((s + 1 < n) ? off[s + 1] : total) - off[s];
}

__global__ void remap_count_kernel(const int64_t *old_off, int64_t n_old, int64_t old_total,
                                   const int64_t *map, int64_t n_new, int64_t *cnt) {
    int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (j >= n_new) return;
    int64_t s = map[j];
    cnt[j] = s < 0 ? 1 : old_seg_len(old_off, n_old, old_total, s);
}

// one warp per new segment, lanes copy the run
__global__ void remap_copy_kernel(const int2 *old_nodes, const int64_t *old_off, int64_t n_old,
                                  int64_t old_total, const int64_t *map, int64_t n_new,
                                  const int64_t *new_off, int2 *new_nodes) {
    int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    int lane = threadIdx.x & 31;
    if (j >= n_new) return;
    int64_t s = map[j];
    int2 *dst = new_nodes + new_off[j];
    if (s < 0) {
        if (lane == 0) dst[0] = make_int2(-1, 0);
        return;
    }
    const int2 *src = old_nodes + old_off[s];
    int64_t len = old_seg_len(old_off, n_old, old_total, s);
    for (int64_t i = lane; i < len; i += 32) dst[i] = src[i];
}

constexpr int kSfPackKt = 4;  // default filters per group (sf_conv.cu supports 4 and 8)

// Fast-stream marking: the last nonzero of every (group, channel) segment gets
// index + kt*9 (its jump-table variant that falls into the channel transition);
// an empty segment's sentinel slot becomes (2*kt*9, run) where run >= 1 counts the
// consecutive empty segments starting at it (the kernel skips a run with one dispatch,
// clipping it to the channel chunk).  Other sentinel slots are never dispatched.
// Row mask of a segment: bit r set iff some nonzero's tap row kh satisfies
// kh <= r <= kh + 3 (the patch rows its FMAs read); a missing segment loads all rows.
__device__ __forceinline__ int seg_row_mask(const int2 *nodes, const int64_t *seg_off, int64_t n_seg,
                                            int64_t total, int64_t t) {
    if (t >= n_seg) return 0x3f;
    const int64_t a = seg_off[t], b = ((t + 1 < n_seg) ? seg_off[t + 1] : total) - 1;
    int m = 0;
    for (int64_t q = a; q < b; ++q) m |= 0xf << ((nodes[q].x % 9) / 3);
    return m;
}

__global__ void sf_pack_mark_kernel(int2 *nodes, const int64_t *seg_off, int64_t n_seg,
                                    int64_t total, int classes) {
    int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (s >= n_seg) return;
    auto seg_len = [&](int64_t t) { return ((t + 1 < n_seg) ? seg_off[t + 1] : total) - seg_off[t]; };
    int64_t start = seg_off[s];
    // read everything this thread needs before anyone rewrites marks (the masks read
    // plain entries; marks only change the index of a segment's last entry, whose
    // kh is the same after % 9, and the sentinel slots, which masks never read)
    if (seg_len(s) == 1) {
        int run = 1;
        while (s + run < n_seg && seg_len(s + run) == 1 && run < (1 << 15)) ++run;
        const int m = seg_row_mask(nodes, seg_off, n_seg, total, s + run);
        nodes[start] = make_int2(2 * classes, run | (m << 16));
    } else {
        const int m = seg_row_mask(nodes, seg_off, n_seg, total, s + 1);
        nodes[start + seg_len(s) - 1].y = m;    // sentinel slot: the next channel's rows
        nodes[start + seg_len(s) - 2].x += classes;
    }
}

}  // namespace

}  // namespace fscnn

using namespace fscnn;

extern "C" {

size_t fscnn_encode_workspace_bytes(int64_t n_segments) {
    return (size_t)(ceil_div(n_segments > 0 ? n_segments : 1, kScanTile) + 1) * sizeof(int64_t);
}

int fscnn_encode_offsets(const float *src, int64_t batch, int64_t outer, int64_t mid,
                         int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                         int64_t *seg_off, int64_t *total_nodes, void *workspace,
                         size_t workspace_bytes, void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    FSCNN_REQUIRE(total_nodes != nullptr, "total_nodes is NULL");
    int64_t n_seg = batch * outer * mid;
    FSCNN_REQUIRE(n_seg == 0 || (src != nullptr || inner == 0) && seg_off != nullptr, "null buffer");
    StridedSrc w{src, outer, mid, inner, s_b, s_o, s_m, s_i, s_o < s_m};
    return encode_offsets_impl(w, n_seg, use_warp_walker(inner, s_i), seg_off, total_nodes,
                               workspace, workspace_bytes, as_stream(stream));
}

int fscnn_encode_nodes(const float *src, int64_t batch, int64_t outer, int64_t mid,
                       int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                       const int64_t *seg_off, fscnn_node *nodes, int64_t *matrix_off,
                       int64_t *tensor_off, void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    int64_t n_seg = batch * outer * mid;
    if (n_seg == 0) return FSCNN_OK;
    FSCNN_REQUIRE(seg_off != nullptr && nodes != nullptr, "null buffer");
    StridedSrc w{src, outer, mid, inner, s_b, s_o, s_m, s_i, s_o < s_m};
    cudaStream_t st = as_stream(stream);
    int rc = FSCNN_OK;
    if (use_tile_writer(w)) {
        const int64_t n_ot = ceil_div(outer, kTO), n_mt = ceil_div(mid, kTM);
        write_tile_kernel<<<(unsigned)(n_ot * n_mt * batch), 256, 0, st>>>(
            w, n_ot, n_mt, seg_off, reinterpret_cast<int2 *>(nodes), -1);
        FSCNN_LAUNCH_CHECK("write_tile_kernel");
    } else {
        rc = encode_nodes_impl(w, n_seg, use_warp_walker(inner, s_i), seg_off, nodes, st);
    }
    if (rc != FSCNN_OK) return rc;
    if (matrix_off || tensor_off) {
        side_tables_kernel<<<(unsigned)ceil_div(n_seg, 256), 256, 0, st>>>(
            seg_off, n_seg, mid, outer * mid, matrix_off, tensor_off);
        FSCNN_LAUNCH_CHECK("side_tables_kernel");
    }
    return FSCNN_OK;
}

int fscnn_decode(const fscnn_node *nodes, const int64_t *seg_off, int64_t batch, int64_t outer,
                 int64_t mid, int64_t inner, float *dst, int64_t d_b, int64_t d_o, int64_t d_m,
                 int64_t d_i, void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    int64_t n_seg = batch * outer * mid;
    if (n_seg == 0 || inner == 0) return FSCNN_OK;
    FSCNN_REQUIRE(nodes && seg_off && dst, "null buffer");
    decode_kernel<<<(unsigned)ceil_div(n_seg, 128), 128, 0, as_stream(stream)>>>(
        reinterpret_cast<const int2 *>(nodes), seg_off, n_seg, outer, mid, inner, dst, nullptr, d_b,
        d_o, d_m, d_i);
    FSCNN_LAUNCH_CHECK("decode_kernel");
    return FSCNN_OK;
}

int fscnn_decode_masked(const fscnn_node *nodes, const int64_t *seg_off, int64_t batch,
                        int64_t outer, int64_t mid, int64_t inner, float *dst, uint8_t *mask,
                        int64_t d_b, int64_t d_o, int64_t d_m, int64_t d_i, void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    int64_t n_seg = batch * outer * mid;
    if (n_seg == 0 || inner == 0) return FSCNN_OK;
    FSCNN_REQUIRE(nodes && seg_off && dst && mask, "null buffer");
    decode_kernel<<<(unsigned)ceil_div(n_seg, 128), 128, 0, as_stream(stream)>>>(
        reinterpret_cast<const int2 *>(nodes), seg_off, n_seg, outer, mid, inner, dst, mask, d_b,
        d_o, d_m, d_i);
    FSCNN_LAUNCH_CHECK("decode_kernel");
    return FSCNN_OK;
}

int fscnn_encode_masked_offsets(const float *src, const uint8_t *mask, int64_t batch,
                                int64_t outer, int64_t mid, int64_t inner, int64_t s_b,
                                int64_t s_o, int64_t s_m, int64_t s_i, int64_t *seg_off,
                                int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                                void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    FSCNN_REQUIRE(total_nodes != nullptr, "total_nodes is NULL");
    int64_t n_seg = batch * outer * mid;
    FSCNN_REQUIRE(n_seg == 0 || ((src && mask) || inner == 0) && seg_off != nullptr, "null buffer");
    MaskedSrc w{src, mask, outer, mid, inner, s_b, s_o, s_m, s_i, s_o < s_m};
    return encode_offsets_impl(w, n_seg, use_warp_walker(inner, s_i), seg_off, total_nodes,
                               workspace, workspace_bytes, as_stream(stream));
}

int fscnn_encode_masked_nodes(const float *src, const uint8_t *mask, int64_t batch,
                              int64_t outer, int64_t mid, int64_t inner, int64_t s_b, int64_t s_o,
                              int64_t s_m, int64_t s_i, const int64_t *seg_off, fscnn_node *nodes,
                              int64_t *matrix_off, int64_t *tensor_off, void *stream) {
    FSCNN_REQUIRE(batch >= 0 && outer >= 0 && mid >= 0 && inner >= 0, "negative extent");
    int64_t n_seg = batch * outer * mid;
    if (n_seg == 0) return FSCNN_OK;
    FSCNN_REQUIRE(seg_off != nullptr && nodes != nullptr, "null buffer");
    MaskedSrc w{src, mask, outer, mid, inner, s_b, s_o, s_m, s_i, s_o < s_m};
    cudaStream_t st = as_stream(stream);
    int rc = encode_nodes_impl(w, n_seg, use_warp_walker(inner, s_i), seg_off, nodes, st);
    if (rc != FSCNN_OK) return rc;
    if (matrix_off || tensor_off) {
        side_tables_kernel<<<(unsigned)ceil_div(n_seg, 256), 256, 0, st>>>(
            seg_off, n_seg, mid, outer * mid, matrix_off, tensor_off);
        FSCNN_LAUNCH_CHECK("side_tables_kernel");
    }
    return FSCNN_OK;
}

int fscnn_remap_segments_offsets(const int64_t *old_seg_off, int64_t n_old, int64_t old_total,
                                 const int64_t *map, int64_t n_new, int64_t *new_seg_off,
                                 int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                                 void *stream) {
    FSCNN_REQUIRE(n_old >= 0 && n_new >= 0 && old_total >= 0, "negative extent");
    FSCNN_REQUIRE(total_nodes != nullptr, "total_nodes is NULL");
    cudaStream_t st = as_stream(stream);
    if (n_new == 0) {
        cudaMemsetAsync(total_nodes, 0, sizeof(int64_t), st);
        return check_launch("memset total");
    }
    FSCNN_REQUIRE(map && new_seg_off && (n_old == 0 || old_seg_off), "null buffer");
    remap_count_kernel<<<(unsigned)ceil_div(n_new, 256), 256, 0, st>>>(old_seg_off, n_old, old_total,
                                                                       map, n_new, new_seg_off);
    FSCNN_LAUNCH_CHECK("remap_count_kernel");
    return scan_inplace(new_seg_off, n_new, total_nodes, workspace, workspace_bytes, st);
}

int fscnn_remap_segments_nodes(const fscnn_node *old_nodes, const int64_t *old_seg_off,
                               int64_t n_old, int64_t old_total, const int64_t *map, int64_t n_new,
                               const int64_t *new_seg_off, fscnn_node *new_nodes, void *stream) {
    FSCNN_REQUIRE(n_old >= 0 && n_new >= 0 && old_total >= 0, "negative extent");
    if (n_new == 0) return FSCNN_OK;
    FSCNN_REQUIRE(map && new_seg_off && new_nodes && (n_old == 0 || (old_nodes && old_seg_off)),
                  "null buffer");
    remap_copy_kernel<<<(unsigned)ceil_div(n_new * 32, 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<const int2 *>(old_nodes), old_seg_off, n_old, old_total, map, n_new,
        new_seg_off, reinterpret_cast<int2 *>(new_nodes));
    FSCNN_LAUNCH_CHECK("remap_copy_kernel");
    return FSCNN_OK;
}

int fscnn_sf_pack_kt(void) { return kSfPackKt; }

int fscnn_sf_pack_offsets(const float *w_kc33, int k, int c, int kt, int64_t *seg_off,
                          int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                          void *stream) {
    FSCNN_REQUIRE(k > 0 && c > 0 && w_kc33 && seg_off && total_nodes, "bad pack arguments");
    FSCNN_REQUIRE(kt == 1 || kt == 2 || kt == 4 || kt == 8, "kt must be 1, 2, 4 or 8");
    int64_t groups = ceil_div(k, kt);
    SfPackSrc src{w_kc33, k, c, kt, (int64_t)kt * 9};
    return encode_offsets_impl(src, groups * c, false, seg_off, total_nodes, workspace,
                               workspace_bytes, as_stream(stream));
}

int fscnn_sf_pack_nodes(const float *w_kc33, int k, int c, int kt, const int64_t *seg_off,
                        int64_t total_nodes, fscnn_node *nodes, void *stream) {
    FSCNN_REQUIRE(k > 0 && c > 0 && w_kc33 && seg_off && nodes, "bad pack arguments");
    FSCNN_REQUIRE(kt == 1 || kt == 2 || kt == 4 || kt == 8, "kt must be 1, 2, 4 or 8");
    int64_t groups = ceil_div(k, kt);
    SfPackSrc src{w_kc33, k, c, kt, (int64_t)kt * 9};
    cudaStream_t st = as_stream(stream);
    int rc = encode_nodes_impl(src, groups * c, false, seg_off, nodes, st, kt * 9);
    if (rc != FSCNN_OK) return rc;
    sf_pack_mark_kernel<<<(unsigned)ceil_div(groups * c, 256), 256, 0, st>>>(
        reinterpret_cast<int2 *>(nodes), seg_off, groups * c, total_nodes, kt * 9);
    FSCNN_LAUNCH_CHECK("sf_pack_mark_kernel");
    return FSCNN_OK;
}

}  // extern "C"
