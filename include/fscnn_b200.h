/*
 * fscnn_b200.h -- C ABI of the B200-native FSCNN sparse-convolution path.
 *
 * Drop-in boundary for the reference package sparse_infer (FSCNN, arXiv 2212.08815).
 * The reference has no native FFI: its operator API is the Python function surface
 * re-exported by sparse_infer/__init__.py:9-74, and each Python wrapper hands flat
 * numpy arrays to one numba kernel.  Every entry point below replaces one of those
 * kernel calls (cited per function) with a stream-ordered launch over DEVICE
 * pointers; INTEGRATION.md shows the ctypes binding a sparse_infer maintainer adds.
 *
 * Conventions (all entry points):
 *   - Pointers are CUDA device pointers; sizes are element counts; strides are in
 *     elements.  `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Node buffers are arrays of fscnn_node, byte-identical to the reference's
 *     NODE_DTYPE = [("index","<i4"),("value","<f4")] (sparse_core.py:24); a node
 *     with index -1 is a segment sentinel with value +0.0.  Offset tables are int64
 *     (sparse_core.py:321-323).
 *   - Dense activations on the device are NCHW float32 ([N][C][H][W]).  The
 *     reference's channel-innermost (W,H,C) DenseTensor3 layout (sparse_core.py:9-13)
 *     is converted at the boundary by fscnn_whc_to_nchw / fscnn_nchw_to_whc.
 *   - Return value: FSCNN_OK or an error code; fscnn_last_error() describes the
 *     last failure on the calling thread.  Validation of shapes and formats is the
 *     caller's (Python) job, as in the reference (kernels are unchecked there too);
 *     the ABI checks only what would make a launch unsafe.
 *   - All kernels are deterministic: results never depend on launch configuration,
 *     batch position or device count (reference contract layers.py:149-155).
 */
#ifndef FSCNN_B200_H
#define FSCNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fscnn_node {
    int32_t index; /* coordinate along the innermost stored axis; -1 = sentinel */
    float value;
} fscnn_node;

enum fscnn_status {
    FSCNN_OK = 0,
    FSCNN_ERR_ARG = 1,         /* bad argument (null pointer, negative extent, ...) */
    FSCNN_ERR_CUDA = 2,        /* a CUDA runtime call or launch failed */
    FSCNN_ERR_UNSUPPORTED = 3  /* geometry not handled by the requested kernel */
};

/* Library identity / diagnostics. */
int fscnn_abi_version(void);
const char *fscnn_last_error(void);
/* Number of kernel launches this library issued since the last reset (host-side counter). */
int64_t fscnn_launch_count(void);
void fscnn_reset_launch_count(void);
/* kernels replayed from a captured CUDA graph (the engine's forward) are not launched
 * through the entry points; the host adds them here so the count stays complete */
void fscnn_add_launch_count(int64_t n);

/* ---------------------------------------------------------------------------
 * Encoder: dense -> node format.
 * Replaces sparsify_tensor3 (sparse_core.py:334-353) with _build_segmented
 * (sparse_core.py:319-331), batched the way SparseTensor4.stack concatenates
 * tensors (sparse_core.py:273-290).
 *
 * The source is viewed as `batch` tensors, each arranged (outer, mid, inner) for
 * the requested axis order; element (b, o, m, i) lives at
 *   src[b*s_b + o*s_o + m*s_m + i*s_i].
 * Segment s = (b*outer + o)*mid + m holds the nonzeros (v != 0.0f: -0.0 dropped,
 * NaN kept) of its inner fiber in ascending i, then one sentinel.
 * seg_off[s] = sum_{t<s} (count[t] + 1)  -- the reference's global offsets.
 *
 * Two calls: fscnn_encode_offsets fills seg_off and *total_nodes (device scalar),
 * the caller sizes the node buffer, then fscnn_encode_nodes writes it.
 * matrix_off (batch*outer, = seg_off[::mid]) and tensor_off (batch) may be NULL.
 * ------------------------------------------------------------------------- */
size_t fscnn_encode_workspace_bytes(int64_t n_segments);
int fscnn_encode_offsets(const float *src, int64_t batch, int64_t outer, int64_t mid,
                         int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                         int64_t *seg_off, int64_t *total_nodes, void *workspace,
                         size_t workspace_bytes, void *stream);
int fscnn_encode_nodes(const float *src, int64_t batch, int64_t outer, int64_t mid,
                       int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                       const int64_t *seg_off, fscnn_node *nodes, int64_t *matrix_off,
                       int64_t *tensor_off, void *stream);

/* Decoder: node format -> dense.  Replaces densify_tensor3 (sparse_core.py:356-368).
 * Writes every element of the strided destination view (zeros where no node). */
int fscnn_decode(const fscnn_node *nodes, const int64_t *seg_off, int64_t batch, int64_t outer,
                 int64_t mid, int64_t inner, float *dst, int64_t d_b, int64_t d_o, int64_t d_m,
                 int64_t d_i, void *stream);

/* Node-preserving variants: decode also writes a presence mask (1 byte per element,
 * same element offsets as dst), and the masked encoder stores an entry iff its mask
 * byte is set, whatever its value.  decode -> masked encode in another axis order is
 * transpose_matrix / transpose_tensor3 (kernels.py:360-411): values, including explicit
 * zero-valued nodes, move untouched. */
int fscnn_decode_masked(const fscnn_node *nodes, const int64_t *seg_off, int64_t batch,
                        int64_t outer, int64_t mid, int64_t inner, float *dst, uint8_t *mask,
                        int64_t d_b, int64_t d_o, int64_t d_m, int64_t d_i, void *stream);
int fscnn_encode_masked_offsets(const float *src, const uint8_t *mask, int64_t batch,
                                int64_t outer, int64_t mid, int64_t inner, int64_t s_b,
                                int64_t s_o, int64_t s_m, int64_t s_i, int64_t *seg_off,
                                int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                                void *stream);
int fscnn_encode_masked_nodes(const float *src, const uint8_t *mask, int64_t batch,
                              int64_t outer, int64_t mid, int64_t inner, int64_t s_b, int64_t s_o,
                              int64_t s_m, int64_t s_i, const int64_t *seg_off, fscnn_node *nodes,
                              int64_t *matrix_off, int64_t *tensor_off, void *stream);

/* Segment gather (node-format restructuring, e.g. pad_tensor on CHW nodes,
 * layers.py:521-535): new segment j is a verbatim copy of old segment map[j] (nodes and
 * sentinel; explicit zero-valued nodes survive) or, for map[j] < 0, an empty segment.
 * Two passes like the encoder: offsets (+ total, workspace as fscnn_encode_*), then
 * nodes.  old_total = length of the old node buffer. */
int fscnn_remap_segments_offsets(const int64_t *old_seg_off, int64_t n_old, int64_t old_total,
                                 const int64_t *map, int64_t n_new, int64_t *new_seg_off,
                                 int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                                 void *stream);
int fscnn_remap_segments_nodes(const fscnn_node *old_nodes, const int64_t *old_seg_off,
                               int64_t n_old, int64_t old_total, const int64_t *map, int64_t n_new,
                               const int64_t *new_seg_off, fscnn_node *new_nodes, void *stream);

/* ---------------------------------------------------------------------------
 * Sparse-Filter convolution, reference order (bit-exact).
 * Replaces _conv_all_filters_kernel (layers.py:170-180) / _conv_filter_sparse_kernel
 * (kernels.py:100-105) over _window_acc (kernels.py:78-97): for every output,
 * taps kw outer, kh inner, nodes ascending c, separate fp32 multiply and add, then
 * + bias[k].  Any geometry (h_f, w_f, stride >= 1, pad >= 0).
 *   x: [n][c][h][w]; nodes/seg_off: CHW SparseTensor4 of K filters, seg_off
 *   [K][w_f*h_f] global; y: [n][K][n_h][n_w]; bias may be NULL (adds +0.0).
 *   relu != 0 applies np.maximum(y, 0) semantics to the result.
 * ------------------------------------------------------------------------- */
int fscnn_sf_conv_exact(const float *x, int n, int c, int h, int w, const fscnn_node *nodes,
                        const int64_t *seg_off, int k, int h_f, int w_f, int stride, int pad,
                        const float *bias, int relu, float *y, void *stream);

/* Dense baseline convolution (bit-exact): conv_forward_dense (layers.py:326-342) over
 * _dense_conv_kernel (kernels.py:169-192) -- taps kh outer, kw inner, channels
 * ascending, every weight multiplied (zeros too, so NaN/Inf inputs propagate as in the
 * reference), then + bias[k].  wt: dense [K][C][h_f][w_f]; x, y as above. */
int fscnn_dense_conv_exact(const float *x, int n, int c, int h, int w, const float *wt, int k,
                           int h_f, int w_f, int stride, int pad, const float *bias, float *y,
                           void *stream);

/* ---------------------------------------------------------------------------
 * Sparse-Filter convolution, fast path (3x3, stride 1, pad 1 -- every VGG16 conv).
 * Same result as fscnn_sf_conv_exact up to fp32 reassociation (channel-major
 * accumulation order).  Consumes the kernel-side packed filter stream:
 *   the filter bank regrouped into groups of `kt` filters; for group g and input
 *   channel c, segment g*c_n + c lists the nonzeros W[g*kt + kl][c][kh][kw] as
 *   nodes with index = kl*9 + kh*3 + kw, ascending, then a sentinel slot.  The last
 *   nonzero of a segment carries index + kt*9 (its jump-table variant that falls into
 *   the channel transition) and an empty segment's sentinel slot carries 2*kt*9
 *   (transition without arithmetic); other sentinel slots are never dispatched.
 * Build it with fscnn_sf_pack_offsets / fscnn_sf_pack_nodes from a dense
 * [K][C][3][3] bank (itself decoded from the reference's CHW SparseTensor4 by
 * fscnn_decode, or straight from dense weights).
 * ------------------------------------------------------------------------- */
int fscnn_sf_pack_kt(void); /* default filters per group (the kernel supports kt = 1, 2, 4 and 8) */
int fscnn_sf_pack_offsets(const float *w_kc33, int k, int c, int kt, int64_t *seg_off,
                          int64_t *total_nodes, void *workspace, size_t workspace_bytes,
                          void *stream);
int fscnn_sf_pack_nodes(const float *w_kc33, int k, int c, int kt, const int64_t *seg_off,
                        int64_t total_nodes, fscnn_node *nodes, void *stream);
/* Fast conv on the HALO-COLUMN layout (not plain NCHW): logical column j of a row
 * lives at memory column j + 1, memory column 0 must be zero (the TMA box that starts
 * one column left of a tile reads it as the left padding) and memory columns > w are
 * never read.  x: [n][c][h][ldi] with ldi >= w + 1, ldi % 4 == 0, 16-byte aligned.
 * y: [n][k][h][ldo] in the same layout -- outputs written at memory columns 1..w,
 * columns 0 and > w left untouched -- or with pool != 0 the fused 2x2 max-pool result
 * [n][k][h/2][ldo] (columns 1..w/2); ldo even and y 8-byte aligned.  A plain NCHW
 * tensor goes in and out with fscnn_pitch_copy (col 0 <-> col 1).  packed/packed_seg_off/total_nodes: the
 * packed stream (allocate total_nodes + 2 nodes: the kernel bulk-copies 16-byte
 * aligned ranges).  max_chunk_entries: the largest node count (sentinels included)
 * of any group over any run of `cc` consecutive channels.  ly selects the
 * sub-region height 4*ly (8, 4 or 2; 0 = by h).  kt: the stream's filters per group
 * (1, 2, 4 or 8) in the low byte; bits 8-15 may ask for 4-warp CTAs with kt = 2 (small
 * grids; 0 = default: 8 warps, 4 for kt = 1) -- the results do not depend on either.  relu applies
 * np.maximum(.,0) before the pool, as the reference's conv -> relu -> pool sequence
 * does. */
int fscnn_sf_conv3x3_ex(const float *x, int n, int c, int h, int w, int ldi,
                        const fscnn_node *packed, const int64_t *packed_seg_off,
                        int64_t total_nodes, int max_chunk_entries, int cc, int k,
                        const float *bias, int relu, int pool, float *y, int ldo, int ly,
                        int kt, void *stream);

/* ---------------------------------------------------------------------------
 * Sparse-Input convolution (bit-exact).
 * Replaces _conv_input_sparse_kernel (kernels.py:136-166) for all K filters at once:
 * output (i,j) of filter k sums, kw outer, kh inner, over the input fiber nodes at
 * (w_in, h_in) ascending c, filt[k][c][kh][kw] * v.  Results that compare equal to
 * 0.0 are written as +0.0 (the reference stores no node for them).
 *   in_nodes: CHW node buffer of n images; in_seg_off: [n][w*h] global offsets
 *   (segment (w_in*h + h_in)); wt: dense filters transposed to [c][kh][kw][K]
 *   (see fscnn_kcrs_to_crsk); y: [n][K][n_h][n_w] (+ bias[k] if bias != NULL).
 * ------------------------------------------------------------------------- */
int fscnn_si_conv(const fscnn_node *in_nodes, const int64_t *in_seg_off, int n, int c, int h,
                  int w, const float *wt, int k, int h_f, int w_f, int stride, int pad,
                  const float *bias, float *y, void *stream);
int fscnn_kcrs_to_crsk(const float *w_kcrs, int k, int c, int r, int s, float *w_crsk,
                       void *stream);
/* 3x3 / stride 1 / pad 1 fast path, same bit-exact results: a warp owns 32 filters and a
 * strip of 8 outputs of one row and walks the strip's input columns left to right (the
 * reference's kw-outer order per output), applying each node to up to three outputs with
 * one 16-byte weight load.  wq: [c][kh][K] float4 {w(kw=0), w(kw=1), w(kw=2), 0} built
 * by fscnn_si_pack3x3 from a dense [K][C][3][3] bank (c*3*K float4 = 48*c*K bytes).
 * The input must satisfy the format's invariant that segments are stored back to back
 * (seg_off[s + 1] == seg_off[s] + count(s) + 1, sentinel last): one-image calls read a
 * fiber's nodes up to seg_off[s + 1] - 1 in coalesced blocks (the Python layer validates
 * this before calling). */
int fscnn_si_pack3x3(const float *w_kc33, int k, int c, float *wq, void *stream);
int fscnn_si_conv3x3(const fscnn_node *in_nodes, const int64_t *in_seg_off, int n, int c, int h,
                     int w, const float *wq, int k, const float *bias, float *y, void *stream);
/* 3x3 / stride 1 / pad 1 channel-major path (the same contraction as
 * _conv_input_sparse_kernel, kernels.py:136-166, summed channel by channel: results
 * within fp32 reassociation of the reference, north-star tolerance max|err| <=
 * 1e-4 max|ref|; deterministic).  K >= 64: a pre-pass merges each output tile's input
 * region fibers into one per-tile channel stream (workspace from the stream-ordered
 * pool: cudaMallocAsync/cudaFreeAsync on `stream`, graph-capturable), then a warp per
 * (tile, filter group) applies every nonzero of a channel with that channel's 9 weights
 * (per filter) held in registers: KT = 4 filters per lane on 4x4 tiles from K = 128,
 * KT = 2 on 4x8 tiles from K = 64; K < 64: one filter per lane, single pass.
 * wf: [c][Kp/(32 KT)][9][32][KT] floats (tap = kh*3+kw, Kp = K padded with zero
 * filters to a multiple of 32 KT, 64 at least), built by fscnn_si_pack_fast from a dense
 * [K][C][3][3] bank; fscnn_si_fast_bank_floats gives its size.  n_nodes: length of
 * in_nodes (bounds the fiber reads and sizes the workspace).  Replaces the same call as
 * fscnn_si_conv3x3 (layers.py:425-428 conv_forward_sparse_input). */
int64_t fscnn_si_fast_bank_floats(int k, int c);
int fscnn_si_pack_fast(const float *w_kc33, int k, int c, float *wf, void *stream);
int fscnn_si_conv3x3_fast(const fscnn_node *in_nodes, const int64_t *in_seg_off, int64_t n_nodes, int n,
                          int c, int h, int w, const float *wf, int k, const float *bias, float *y,
                          void *stream);
/* Same with Alg. 7's pooling fused into the epilogue (layers.py:345-390): pool = 1 for a
 * 2x2 max-pool, 2 for a 2x2 average-pool, applied to the conv output in
 * _pool_dense_kernel's order (layers.py:250-271; as fscnn_pool2d) before + bias;
 * y is [n][k][h/2][w/2] (h, w even).  pool = 0 is fscnn_si_conv3x3_fast. */
int fscnn_si_conv3x3_fast_pool(const fscnn_node *in_nodes, const int64_t *in_seg_off, int64_t n_nodes, int n,
                               int c, int h, int w, const float *wf, int k, const float *bias, int pool,
                               float *y, void *stream);
/* The same conv (pool as above) straight from a dense activation x [n][c][h][w] (fp32,
 * contiguous) instead of its CHW node encoding -- the result is bit-identical to
 * encoding x (fscnn_encode_*: values +-0.0 not stored, NaN stored) and calling
 * fscnn_si_conv3x3_fast_pool: the tile streams hold the same entries.  K >= 64.  Lets a
 * stack of sparse-input layers skip the re-encode (count, scan, host sync, write)
 * between layers. */
int fscnn_si_conv3x3_fast_dense(const float *x, int n, int c, int h, int w, const float *wf, int k,
                                const float *bias, int pool, float *y, void *stream);

/* ---------------------------------------------------------------------------
 * Dense layers between convolutions.
 *   fscnn_relu: np.maximum(x, 0) semantics (layers.py:469-484): NaN propagates,
 *     -0.0 -> +0.0.
 *   fscnn_pool2d: _pool_dense_kernel (layers.py:250-271) on NCHW: non-overlapping
 *     (h_p, w_p) windows; max: -inf start, take v iff v > acc (ph outer, pw inner);
 *     avg: same-order sum / (h_p*w_p).
 *   Layout converters between the reference's (W,H,C) DenseTensor3 memory and NCHW.
 * ------------------------------------------------------------------------- */
int fscnn_relu(const float *x, int64_t count, float *y, void *stream);
/* kind 0 = fscnn_relu; 1 = leaky ReLU np.where(x > 0, x, slope*x) (layers.py:484);
 * 2 = the node-format ReLU keep rule x > 0 ? x : 0 (layers.py:488-489, with
 * rebuild_tensor3 sparse_core.py:460-473 done by decode -> this -> re-encode). */
int fscnn_activation(const float *x, int64_t count, int kind, float slope, float *y,
                     void *stream);
/* apply_batchnorm (layers.py:507-509) on NCHW: ((x - mean) / sqrt(var + eps)) * scale + shift
 * with numpy's float32 op order (bit-exact). */
int fscnn_batchnorm(const float *x, int n, int c, int h, int w, const float *scale,
                    const float *shift, const float *mean, const float *var, float eps, float *y,
                    void *stream);
/* pad_tensor (layers.py:513-520) on NCHW: y is (h + 2p) x (w + 2p), zeros around. */
int fscnn_pad2d(const float *x, int n, int c, int h, int w, int p, float *y, void *stream);
int fscnn_pool2d(const float *x, int n, int c, int h, int w, int h_p, int w_p, int use_max,
                 float *y, void *stream);
int fscnn_whc_to_nchw(const float *x_whc, int n, int c, int h, int w, float *y_nchw,
                      void *stream);
int fscnn_nchw_to_whc(const float *x_nchw, int n, int c, int h, int w, float *y_whc,
                      void *stream);
/* Pitched variants: the NCHW side has row pitch ld (floats) and its rows start at column
 * col0 -- (ld, col0) = (halo_pitch(w), 1) reads/writes the fast kernel's halo-column
 * layout directly, so the public-API forward stages and unstages in one pass each. */
int fscnn_whc_to_nchw_ex(const float *x_whc, int n, int c, int h, int w, float *y, int ld,
                         int col0, void *stream);
int fscnn_nchw_to_whc_ex(const float *x, int n, int c, int h, int w, int ld, int col0, float *y_whc,
                         void *stream);

/* FP32 CUDA-core throughput probe (roofline denominator): `blocks` x 256 threads,
 * each 8 independent FFMA chains of 16*iters steps = 256*blocks*iters*256 FLOPs. */
/* Per-layer specialised sparse-filter 3x3/s1/p1 conv (+bias, ReLU, fused 2x2 max-pool):
 * the bank's nonzero pattern and values are compiled into the kernel (one straight-line
 * kernel per group of up to 32 filters, weights as FFMA2 immediates; PTX generated here,
 * compiled with nvJitLink on host threads, cached on disk by content hash).  Replaces
 * the same reference routine as fscnn_sf_conv3x3_ex -- _conv_all_filters_kernel
 * (layers.py:170-180) over _window_acc (kernels.py:78-97) -- with the same accumulation
 * order, so its outputs are bit-identical to fscnn_sf_conv3x3_ex's.
 *   create: w_kc33 = dense host bank [k][c][3][3] (+-0.0 entries are absent nodes),
 *           bias = host [k] or NULL; h, w even; flags: bits 0-7 filters per group
 *           (0 = 48), bits 8-15 a cap on warps per CTA (0 = none), bit 16: one fused
 *           kernel for all groups (small layers: one launch).  Returns immediately: the
 *           compile runs in the background; wait (or the first launch) joins it.
 *   launch: x = halo-column input [n][c][h][ldi] (logical column j at memory column j+1,
 *           column 0 zero, ldi >= w+1 and a multiple of 4, 16-byte aligned);
 *           y = halo-column output [n][k][h'][ldo] (h' = h/2, w' = w/2 with the pool;
 *           columns 0 and > w' of y are not written). */
typedef struct fscnn_sfjit fscnn_sfjit;
int fscnn_sfjit_create(const float *w_kc33, const float *bias, int k, int c, int h, int w, int relu,
                       int pool, int flags, fscnn_sfjit **out);
int fscnn_sfjit_compiled(fscnn_sfjit *j); /* join the compile jobs (no GPU needed) */
int fscnn_sfjit_wait(fscnn_sfjit *j);     /* compiled + modules loaded in the current context */
int fscnn_sfjit_launch(fscnn_sfjit *j, const float *x, int n, int ldi, float *y, int ldo, void *stream);
int fscnn_sfjit_info(fscnn_sfjit *j, int64_t *info, double *secs);
void fscnn_sfjit_destroy(fscnn_sfjit *j);
/* PTX of one group (inspection, CPU tests): length, copied into buf when cap > length. */
int64_t fscnn_sfjit_ptx(const float *w_kc33, const float *bias, int k, int c, int h, int w, int relu,
                        int pool, int flags, int group, char *buf, int64_t cap);

/* Row-pitched copy of `rows` rows of w floats: y[r*ldy + coly + j] = x[r*ldx + colx + j].
 * Dense NCHW <-> the halo-column activation layout (no reference counterpart: staging
 * around the conv stack of network.py:410-534). */
int fscnn_pitch_copy(const float *x, int64_t rows, int w, int ldx, int colx, float *y, int ldy,
                     int coly, void *stream);

int fscnn_fp32_probe(float *out, int blocks, int iters, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* FSCNN_B200_H */
