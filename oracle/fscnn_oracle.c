/*
 * fscnn_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference sparse_infer hot path (FSCNN, arXiv 2212.08815),
 * used as the parity checker by tests/, __graft_entry__.smoke() and as bench.py's
 * cpu_baseline / `--impl reference` leg.  Nothing in the product package links,
 * imports or executes this file.
 *
 * Every function restates one reference routine loop-for-loop (same accumulation
 * order, separate float32 multiply and add -- built with -ffp-contract=off so the
 * compiler cannot fuse them, matching numba's default non-fastmath lowering).
 * Parity of this restatement is pinned against golden vectors produced by the
 * reference itself (tests/golden/make_golden.py -> tests/golden/*.npz).
 *
 * Layout conventions are the reference's own:
 *   dense 3-D tensor (C,H,W): element (c,h,w) at (w*H + h)*C + c  (sparse_core.py:9-13)
 *   node: {int32 index, float32 value}, sentinel index -1      (sparse_core.py:24)
 *   all offset tables int64                                     (sparse_core.py:321-323)
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int32_t index;
    float value;
} node_t;

static void set_threads(int n_threads) {
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#else
    (void)n_threads;
#endif
}

int oracle_has_openmp(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 0;
#endif
}

/* ---------------------------------------------------------------------------
 * Encoder.  Restates sparse_core.py:319-331 (_build_segmented) driven by the
 * np.nonzero scan of sparsify_tensor3 (sparse_core.py:334-353): the arranged
 * (outer, mid, inner) view is scanned row-major, segment id = outer*mid + mid,
 * offsets[s] = sum_{t<s}(count[t] + 1), each segment's entries in scan order,
 * then one sentinel (-1, +0.0).  A value is "nonzero" iff v != 0.0f, so -0.0
 * is dropped and NaN is kept (np.nonzero semantics).
 *
 * Generalised to a batch: segment s = (b*outer + o)*mid + m, source element
 * address = b*s_b + o*s_o + m*s_m + i*s_i.  The batch concatenation matches
 * SparseTensor4.stack (sparse_core.py:273-290): global offsets are the running
 * sum over all earlier tensors.
 * ------------------------------------------------------------------------- */
int64_t oracle_encode_count(const float *src, int64_t batch, int64_t outer, int64_t mid,
                            int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                            int64_t *seg_off) {
    int64_t pos = 0;
    int64_t s = 0;
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t o = 0; o < outer; ++o)
            for (int64_t m = 0; m < mid; ++m, ++s) {
                const float *row = src + b * s_b + o * s_o + m * s_m;
                int64_t cnt = 0;
                for (int64_t i = 0; i < inner; ++i)
                    if (row[i * s_i] != 0.0f) ++cnt;
                seg_off[s] = pos;
                pos += cnt + 1;
            }
    return pos;
}

void oracle_encode_write(const float *src, int64_t batch, int64_t outer, int64_t mid,
                         int64_t inner, int64_t s_b, int64_t s_o, int64_t s_m, int64_t s_i,
                         const int64_t *seg_off, node_t *nodes) {
    int64_t s = 0;
    for (int64_t b = 0; b < batch; ++b)
        for (int64_t o = 0; o < outer; ++o)
            for (int64_t m = 0; m < mid; ++m, ++s) {
                const float *row = src + b * s_b + o * s_o + m * s_m;
                int64_t p = seg_off[s];
                for (int64_t i = 0; i < inner; ++i) {
                    float v = row[i * s_i];
                    if (v != 0.0f) {
                        nodes[p].index = (int32_t)i;
                        nodes[p].value = v;
                        ++p;
                    }
                }
                nodes[p].index = -1;
                nodes[p].value = 0.0f;
            }
}

/* Decoder: restates densify_tensor3 (sparse_core.py:356-368) for one arranged
 * view -- every data node of segment s lands at (s, index); the rest is zero. */
void oracle_decode(const node_t *nodes, const int64_t *seg_off, int64_t n_seg, int64_t inner,
                   float *dst /* n_seg x inner, zero-initialised by caller */) {
    for (int64_t s = 0; s < n_seg; ++s) {
        int64_t p = seg_off[s];
        while (nodes[p].index != -1) {
            dst[s * inner + nodes[p].index] = nodes[p].value;
            ++p;
        }
    }
}

/* ---------------------------------------------------------------------------
 * Sparse-Filter convolution.  Restates _window_acc (kernels.py:78-97) inside
 * _conv_all_filters_kernel (layers.py:170-180): for output (w, h, f),
 *   x = 0; for l in W_F: for k in H_F: for node in segment(f, l*H_F + k): x += in*val
 *   out[w, h, f] = x + bias[f]
 * Padding is virtual (out-of-range taps skipped).  Input and output are the
 * reference's channel-innermost (W, H, C) layout, one image after another.
 * seg_off is the SparseTensor4 global segment table (K x H_F*W_F, int64).
 * Parallel over (image, output column, output row) -- results do not depend on threads.
 * ------------------------------------------------------------------------- */
static float window_acc(const float *inp, int h_i, int w_i, int c_n, const node_t *nodes,
                        const int64_t *seg_off, int64_t seg_base, int w_f, int h_f, int w0,
                        int h0) {
    float x = 0.0f;
    for (int l = 0; l < w_f; ++l) {
        int w_in = l + w0;
        if (w_in < 0 || w_in >= w_i) continue;
        int64_t col = seg_base + (int64_t)l * h_f;
        for (int k = 0; k < h_f; ++k) {
            int h_in = k + h0;
            if (h_in < 0 || h_in >= h_i) continue;
            const float *fib = inp + ((int64_t)w_in * h_i + h_in) * c_n;
            int64_t p = seg_off[col + k];
            while (nodes[p].index != -1) {
                float prod = fib[nodes[p].index] * nodes[p].value;
                x = x + prod;
                ++p;
            }
        }
    }
    return x;
}

void oracle_sf_conv(const float *inp, int64_t n_img, int c_n, int h_i, int w_i,
                    const node_t *nodes, const int64_t *seg_off, int k_n, int h_f, int w_f,
                    int stride, int pad, const float *bias, float *out, int n_threads) {
    int n_h = (h_i + 2 * pad - h_f) / stride + 1;
    int n_w = (w_i + 2 * pad - w_f) / stride + 1;
    int64_t in_sz = (int64_t)c_n * h_i * w_i;
    int64_t out_sz = (int64_t)k_n * n_h * n_w;
    set_threads(n_threads);
#pragma omp parallel for collapse(3) schedule(dynamic, 4)
    for (int64_t img = 0; img < n_img; ++img)
        for (int w = 0; w < n_w; ++w)
            for (int h = 0; h < n_h; ++h) {
                const float *in_img = inp + img * in_sz;
                float *o = out + img * out_sz;
                for (int f = 0; f < k_n; ++f) {
                    float x = window_acc(in_img, h_i, w_i, c_n, nodes, seg_off,
                                         (int64_t)f * h_f * w_f, w_f, h_f, w * stride - pad,
                                         h * stride - pad);
                    float b = bias ? bias[f] : 0.0f;
                    o[((int64_t)w * n_h + h) * k_n + f] = x + b;
                }
        }
}

/* Exact multiply tally of _conv_filter_sparse_counted_kernel (kernels.py:108-133):
 * per filter, sum over in-bounds taps of the tap segment's node count.  The
 * reported nnz-FLOPs are 2x this. */
int64_t oracle_sf_count(int h_i, int w_i, const int64_t *seg_off, int64_t n_nodes, int k_n,
                        int h_f, int w_f, int stride, int pad) {
    int n_h = (h_i + 2 * pad - h_f) / stride + 1;
    int n_w = (w_i + 2 * pad - w_f) / stride + 1;
    int64_t total = 0;
    int64_t n_seg = (int64_t)k_n * h_f * w_f;
    for (int64_t s = 0; s < n_seg; ++s) {
        int64_t end = (s + 1 < n_seg) ? seg_off[s + 1] : n_nodes;
        int64_t nnz = end - seg_off[s] - 1;
        int tap = (int)(s % (h_f * w_f));
        int l = tap / h_f, k = tap % h_f;
        int64_t rows = 0, cols = 0;
        for (int i = 0; i < n_h; ++i) {
            int h_in = k + i * stride - pad;
            rows += (h_in >= 0 && h_in < h_i);
        }
        for (int j = 0; j < n_w; ++j) {
            int w_in = l + j * stride - pad;
            cols += (w_in >= 0 && w_in < w_i);
        }
        total += nnz * rows * cols;
    }
    return total;
}

/* ---------------------------------------------------------------------------
 * Sparse-Input convolution.  Restates _conv_input_sparse_kernel
 * (kernels.py:136-166): for output (i, j) of filter f,
 *   x = 0; for l in W_F: for k in H_F: for node in fiber(w_in*H_I + h_in): x += filt[l,k,c]*v
 * The reference appends x only when x != 0.0; its densified form (densify_matrix)
 * therefore holds +0.0 wherever x compared equal to zero -- reproduced here.
 * filt: K filters, each (W_F, H_F, C) channel-innermost (DenseTensor3 data).
 * in_seg_off: per-image CHW segment table (H_I*W_I entries, image-local offsets),
 * images' node buffers at in_nodes + node_base[img].
 * Output: dense (K, n_h, n_w) per image, image after image.
 * ------------------------------------------------------------------------- */
void oracle_si_conv(const node_t *in_nodes, const int64_t *node_base, const int64_t *in_seg_off,
                    int64_t n_img, int c_n, int h_i, int w_i, const float *filt, int k_n, int h_f,
                    int w_f, int stride, int pad, float *out, int n_threads) {
    int n_h = (h_i + 2 * pad - h_f) / stride + 1;
    int n_w = (w_i + 2 * pad - w_f) / stride + 1;
    int64_t f_sz = (int64_t)w_f * h_f * c_n;
    int64_t out_sz = (int64_t)k_n * n_h * n_w;
    set_threads(n_threads);
#pragma omp parallel for collapse(2) schedule(dynamic, 1)
    for (int64_t img = 0; img < n_img; ++img)
        for (int f = 0; f < k_n; ++f) {
            const node_t *nd = in_nodes + node_base[img];
            const int64_t *so = in_seg_off + img * (int64_t)h_i * w_i;
            const float *fl = filt + f * f_sz;
            float *o = out + img * out_sz + (int64_t)f * n_h * n_w;
            for (int i = 0; i < n_h; ++i)
                for (int j = 0; j < n_w; ++j) {
                    float x = 0.0f;
                    for (int l = 0; l < w_f; ++l) {
                        int w_in = l + j * stride - pad;
                        if (w_in < 0 || w_in >= w_i) continue;
                        for (int k = 0; k < h_f; ++k) {
                            int h_in = k + i * stride - pad;
                            if (h_in < 0 || h_in >= h_i) continue;
                            int64_t q = so[(int64_t)w_in * h_i + h_in];
                            while (nd[q].index != -1) {
                                float prod = fl[((int64_t)l * h_f + k) * c_n + nd[q].index] *
                                             nd[q].value;
                                x = x + prod;
                                ++q;
                            }
                        }
                    }
                    o[(int64_t)i * n_w + j] = (x != 0.0f) ? x : 0.0f;
                }
        }
}

/* ---------------------------------------------------------------------------
 * Dense cross-correlation oracle.  Restates _dense_conv_kernel
 * (kernels.py:169-192): accumulation order (k, l, c).  Output (K, n_h, n_w).
 * ------------------------------------------------------------------------- */
void oracle_dense_conv(const float *inp, int c_n, int h_i, int w_i, const float *filt, int k_n,
                       int h_f, int w_f, int stride, int pad, float *out, int n_threads) {
    int n_h = (h_i + 2 * pad - h_f) / stride + 1;
    int n_w = (w_i + 2 * pad - w_f) / stride + 1;
    int64_t f_sz = (int64_t)w_f * h_f * c_n;
    set_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 1)
    for (int f = 0; f < k_n; ++f) {
        const float *fl = filt + f * f_sz;
        for (int i = 0; i < n_h; ++i)
            for (int j = 0; j < n_w; ++j) {
                float x = 0.0f;
                for (int k = 0; k < h_f; ++k) {
                    int h_in = k + i * stride - pad;
                    if (h_in < 0 || h_in >= h_i) continue;
                    for (int l = 0; l < w_f; ++l) {
                        int w_in = l + j * stride - pad;
                        if (w_in < 0 || w_in >= w_i) continue;
                        const float *fib = inp + ((int64_t)w_in * h_i + h_in) * c_n;
                        const float *wf = fl + ((int64_t)l * h_f + k) * c_n;
                        for (int c = 0; c < c_n; ++c) {
                            float prod = fib[c] * wf[c];
                            x = x + prod;
                        }
                    }
                }
                out[((int64_t)f * n_h + i) * n_w + j] = x;
            }
    }
}

/* ---------------------------------------------------------------------------
 * Pooling.  Restates _pool_dense_kernel (layers.py:250-271): non-overlapping
 * windows; max starts at -inf and takes v only if v > acc (ph outer, pw inner);
 * avg sums in the same order and divides by the float32 area.
 * Layout (W, H, C) in and out, image after image.
 * ------------------------------------------------------------------------- */
void oracle_pool(const float *inp, int64_t n_img, int c_n, int h, int w, int h_p, int w_p,
                 int use_max, float *out) {
    int h_o = h / h_p, w_o = w / w_p;
    float area = (float)(h_p * w_p);
    for (int64_t img = 0; img < n_img; ++img) {
        const float *in_img = inp + img * (int64_t)c_n * h * w;
        float *o = out + img * (int64_t)c_n * h_o * w_o;
        for (int wo = 0; wo < w_o; ++wo)
            for (int ho = 0; ho < h_o; ++ho)
                for (int c = 0; c < c_n; ++c) {
                    float acc = use_max ? -INFINITY : 0.0f;
                    for (int ph = 0; ph < h_p; ++ph)
                        for (int pw = 0; pw < w_p; ++pw) {
                            float v = in_img[((int64_t)(wo * w_p + pw) * h + (ho * h_p + ph)) * c_n + c];
                            if (use_max) {
                                if (v > acc) acc = v;
                            } else {
                                acc = acc + v;
                            }
                        }
                    o[((int64_t)wo * h_o + ho) * c_n + c] = use_max ? acc : acc / area;
                }
    }
}

/* ReLU as np.maximum(x, 0.0f) (layers.py:482-483): NaN propagates; otherwise the
 * first operand wins only if strictly greater, so -0.0 becomes +0.0. */
void oracle_relu(const float *inp, int64_t n, float *out) {
    for (int64_t i = 0; i < n; ++i) {
        float v = inp[i];
        out[i] = (v > 0.0f || isnan(v)) ? v : 0.0f;
    }
}

/* ---------------------------------------------------------------------------
 * Node-format activations.  Restates apply_activation's SparseTensor3 branch
 * (layers.py:485-491) over rebuild_tensor3 (sparse_core.py:460-473): walk every
 * segment's data nodes in buffer order; kind 0 (ReLU) keeps a node iff value > 0
 * (value unchanged), kind 1 (LeakyReLU) maps v -> (v > 0 ? v : slope * v) and keeps
 * the node iff the new value != 0; every segment ends with a sentinel; offsets are
 * the running sum of (kept + 1).  out == NULL: count only.  Returns the node total.
 * ------------------------------------------------------------------------- */
int64_t oracle_rebuild(const node_t *nodes, const int64_t *seg_off, int64_t n_seg, int kind,
                       float slope, int64_t *new_off, node_t *out) {
    int64_t pos = 0;
    for (int64_t s = 0; s < n_seg; ++s) {
        new_off[s] = pos;
        for (int64_t p = seg_off[s]; nodes[p].index != -1; ++p) {
            float v = nodes[p].value, nv = v;
            int keep;
            if (kind == 0) {
                keep = v > 0.0f;
            } else {
                nv = v > 0.0f ? v : slope * v;
                keep = nv != 0.0f;
            }
            if (keep) {
                if (out) {
                    out[pos].index = nodes[p].index;
                    out[pos].value = nv;
                }
                ++pos;
            }
        }
        if (out) {
            out[pos].index = -1;
            out[pos].value = 0.0f;
        }
        ++pos;
    }
    return pos;
}

/* Batch norm, inference (layers.py:507-509) on a (W, H, C) payload:
 * ((x - mean[c]) / sqrt(var[c] + eps)) * scale[c] + shift[c], float32 throughout. */
void oracle_batchnorm(const float *inp, int c_n, int64_t hw, const float *scale, const float *shift,
                      const float *mean, const float *var, float eps, float *out) {
    for (int64_t q = 0; q < hw; ++q)
        for (int c = 0; c < c_n; ++c) {
            float sd = sqrtf(var[c] + eps);
            out[q * c_n + c] = ((inp[q * c_n + c] - mean[c]) / sd) * scale[c] + shift[c];
        }
}

/* pad_tensor, dense (layers.py:518-520): (W, H, C) -> (W+2p, H+2p, C), zeros around. */
void oracle_pad_dense(const float *inp, int c_n, int h, int w, int p, float *out) {
    int hp = h + 2 * p, wp = w + 2 * p;
    for (int x = 0; x < wp; ++x)
        for (int y = 0; y < hp; ++y)
            for (int c = 0; c < c_n; ++c) {
                int xi = x - p, yi = y - p;
                out[((int64_t)x * hp + y) * c_n + c] =
                    (xi >= 0 && xi < w && yi >= 0 && yi < h) ? inp[((int64_t)xi * h + yi) * c_n + c] : 0.0f;
            }
}

/* pad_tensor, CHW nodes (layers.py:521-535): channel fibers keep their nodes; segment
 * (w*H + h) moves to ((w+p)*(H+2p) + h+p); new border segments are empty.
 * out == NULL: offsets only.  Returns the node total. */
int64_t oracle_pad_chw_nodes(const node_t *nodes, const int64_t *seg_off, int h, int w, int p,
                             int64_t *new_off, node_t *out) {
    int hp = h + 2 * p, wp = w + 2 * p;
    int64_t pos = 0;
    for (int x = 0; x < wp; ++x)
        for (int y = 0; y < hp; ++y) {
            int64_t s = (int64_t)x * hp + y;
            new_off[s] = pos;
            int xi = x - p, yi = y - p;
            if (xi >= 0 && xi < w && yi >= 0 && yi < h) {
                for (int64_t q = seg_off[(int64_t)xi * h + yi]; nodes[q].index != -1; ++q) {
                    if (out) out[pos] = nodes[q];
                    ++pos;
                }
            }
            if (out) {
                out[pos].index = -1;
                out[pos].value = 0.0f;
            }
            ++pos;
        }
    return pos;
}

/* transpose_matrix (kernels.py:360-380 over _transpose_segments_kernel :195-223):
 * re-bucket n_seg segments by node index into seg_len new segments -- counts, running
 * offsets (count + 1), scatter in buffer order with new index = old segment id, then
 * the sentinels.  Values move untouched.  Returns the node total. */
int64_t oracle_transpose_segments(const node_t *nodes, int64_t total, int64_t seg_len,
                                  int64_t *new_off, node_t *out, int64_t *cursor /* seg_len */) {
    for (int64_t i = 0; i < seg_len; ++i) cursor[i] = 0;
    for (int64_t p = 0; p < total; ++p)
        if (nodes[p].index != -1) ++cursor[nodes[p].index];
    int64_t pos = 0;
    for (int64_t i = 0; i < seg_len; ++i) {
        new_off[i] = pos;
        int64_t cnt = cursor[i];
        cursor[i] = pos;
        pos += cnt + 1;
    }
    int32_t seg = 0;
    for (int64_t p = 0; p < total; ++p) {
        if (nodes[p].index == -1) {
            ++seg;
        } else {
            int64_t at = cursor[nodes[p].index]++;
            out[at].index = seg;
            out[at].value = nodes[p].value;
        }
    }
    for (int64_t i = 0; i < seg_len; ++i) {
        out[cursor[i]].index = -1;
        out[cursor[i]].value = 0.0f;
    }
    return pos;
}

/* transpose_tensor3 WHC -> CHW (kernels.py:383-411): node (c, h, w, v) of segment
 * (c*H + h) at index w moves to segment (w*H + h) at index c; new segments list their
 * nodes with c ascending (the reference's per-channel re-bucket + (w, h, c) gather).
 * Returns the node total. */
int64_t oracle_transpose_whc_to_chw(const node_t *nodes, const int64_t *seg_off, int c_n, int h,
                                    int w, int64_t *new_off, node_t *out, int64_t *cursor /* w*h */) {
    int64_t n_new = (int64_t)w * h;
    for (int64_t s = 0; s < n_new; ++s) cursor[s] = 0;
    for (int c = 0; c < c_n; ++c)
        for (int y = 0; y < h; ++y)
            for (int64_t q = seg_off[(int64_t)c * h + y]; nodes[q].index != -1; ++q)
                ++cursor[(int64_t)nodes[q].index * h + y];
    int64_t pos = 0;
    for (int64_t s = 0; s < n_new; ++s) {
        new_off[s] = pos;
        int64_t cnt = cursor[s];
        cursor[s] = pos;
        pos += cnt + 1;
    }
    for (int c = 0; c < c_n; ++c)
        for (int y = 0; y < h; ++y)
            for (int64_t q = seg_off[(int64_t)c * h + y]; nodes[q].index != -1; ++q) {
                int64_t at = cursor[(int64_t)nodes[q].index * h + y]++;
                out[at].index = c;
                out[at].value = nodes[q].value;
            }
    for (int64_t s = 0; s < n_new; ++s) {
        out[cursor[s]].index = -1;
        out[cursor[s]].value = 0.0f;
    }
    return pos;
}
