"""TEST INFRASTRUCTURE ONLY -- ctypes front of the CPU restatement (fscnn_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module.  It is the checker (and the CPU baseline), never the
product: the package paper_2212_08815_b200 does not import it.

Every routine here drives one C function that restates a reference routine; the
docstrings name the reference file:line.  Arrays use the reference's own layouts:
dense 3-D tensors are channel-innermost (W, H, C) memory, node buffers are the
8-byte {int32 index, float32 value} records of sparse_core.NODE_DTYPE.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

NODE_DTYPE = np.dtype([("index", "<i4"), ("value", "<f4")])

# (inner, mid, outer) axis ids, 0=C 1=H 2=W, per order name (sparse_core.py:44-66)
ORDER_AXES = {
    "WHC": (2, 1, 0),
    "WCH": (2, 0, 1),
    "HWC": (1, 2, 0),
    "HCW": (1, 0, 2),
    "CHW": (0, 1, 2),
    "CWH": (0, 2, 1),
}

_lib = None


def build() -> str:
    """Compile liboracle.so with the committed Makefile (idempotent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        L.oracle_encode_count.restype = i64
        L.oracle_encode_count.argtypes = [vp] + [i64] * 8 + [vp]
        L.oracle_encode_write.restype = None
        L.oracle_encode_write.argtypes = [vp] + [i64] * 8 + [vp, vp]
        L.oracle_decode.restype = None
        L.oracle_decode.argtypes = [vp, vp, i64, i64, vp]
        L.oracle_sf_conv.restype = None
        L.oracle_sf_conv.argtypes = [vp, i64, i32, i32, i32, vp, vp, i32, i32, i32, i32, i32, vp, vp, i32]
        L.oracle_sf_count.restype = i64
        L.oracle_sf_count.argtypes = [i32, i32, vp, i64, i32, i32, i32, i32, i32]
        L.oracle_si_conv.restype = None
        L.oracle_si_conv.argtypes = [vp, vp, vp, i64, i32, i32, i32, vp, i32, i32, i32, i32, i32, vp, i32]
        L.oracle_dense_conv.restype = None
        L.oracle_dense_conv.argtypes = [vp, i32, i32, i32, vp, i32, i32, i32, i32, i32, vp, i32]
        L.oracle_pool.restype = None
        L.oracle_pool.argtypes = [vp, i64, i32, i32, i32, i32, i32, i32, vp]
        L.oracle_relu.restype = None
        L.oracle_relu.argtypes = [vp, i64, vp]
        L.oracle_has_openmp.restype = i32
        f32 = ctypes.c_float
        L.oracle_rebuild.restype = i64
        L.oracle_rebuild.argtypes = [vp, vp, i64, i32, f32, vp, vp]
        L.oracle_batchnorm.restype = None
        L.oracle_batchnorm.argtypes = [vp, i32, i64, vp, vp, vp, vp, f32, vp]
        L.oracle_pad_dense.restype = None
        L.oracle_pad_dense.argtypes = [vp, i32, i32, i32, i32, vp]
        L.oracle_pad_chw_nodes.restype = i64
        L.oracle_pad_chw_nodes.argtypes = [vp, vp, i32, i32, i32, vp, vp]
        L.oracle_transpose_segments.restype = i64
        L.oracle_transpose_segments.argtypes = [vp, i64, i64, vp, vp, vp]
        L.oracle_transpose_whc_to_chw.restype = i64
        L.oracle_transpose_whc_to_chw.argtypes = [vp, vp, i32, i32, i32, vp, vp, vp]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def max_threads() -> int:
    return max(1, int(lib().oracle_has_openmp()))


# -- encoder / decoder -----------------------------------------------------------


def encode_batch(arrs_chw: np.ndarray, order: str = "CHW"):
    """Encode a batch of (C, H, W)-indexed arrays in ``order``.

    Restates sparsify_tensor3 (sparse_core.py:334-353) for each tensor and the
    concatenation of SparseTensor4.stack (sparse_core.py:273-290).  Returns
    (nodes, tensor_offsets[B], matrix_offsets[B, outer], segment_offsets[B, outer*mid]).
    """
    a = np.ascontiguousarray(arrs_chw, dtype=np.float32)
    if a.ndim == 3:
        a = a[None]
    b_n = a.shape[0]
    inner_ax, mid_ax, outer_ax = ORDER_AXES[order]
    dims = a.shape[1:]
    es = [s // 4 for s in a.strides]  # element strides: b, c, h, w
    inner, mid, outer = dims[inner_ax], dims[mid_ax], dims[outer_ax]
    s_b = es[0]
    s_i, s_m, s_o = es[1 + inner_ax], es[1 + mid_ax], es[1 + outer_ax]
    n_seg = b_n * outer * mid
    seg = np.empty(n_seg, np.int64)
    L = lib()
    total = L.oracle_encode_count(_p(a), b_n, outer, mid, inner, s_b, s_o, s_m, s_i, _p(seg))
    nodes = np.empty(total, NODE_DTYPE)
    L.oracle_encode_write(_p(a), b_n, outer, mid, inner, s_b, s_o, s_m, s_i, _p(seg), _p(nodes))
    seg2 = seg.reshape(b_n, outer * mid)
    return nodes, seg2[:, 0].copy(), np.ascontiguousarray(seg2[:, ::mid]), seg2


def encode(arr_chw: np.ndarray, order: str = "CHW"):
    """One tensor: (nodes, matrix_offsets, segment_offsets) as sparsify_tensor3 makes them."""
    nodes, _, mat, seg = encode_batch(np.asarray(arr_chw)[None], order)
    return nodes, mat[0].copy(), seg[0].copy()


def decode(nodes: np.ndarray, seg_off: np.ndarray, dims_chw, order: str = "CHW") -> np.ndarray:
    """Restates densify_tensor3 (sparse_core.py:356-368); returns the (C, H, W) array."""
    inner_ax, mid_ax, outer_ax = ORDER_AXES[order]
    inner, mid, outer = dims_chw[inner_ax], dims_chw[mid_ax], dims_chw[outer_ax]
    arranged = np.zeros((outer, mid, inner), np.float32)
    nodes = np.ascontiguousarray(nodes)
    seg = np.ascontiguousarray(seg_off, dtype=np.int64)
    lib().oracle_decode(_p(nodes), _p(seg), outer * mid, inner, _p(arranged))
    perm = [(outer_ax, mid_ax, inner_ax).index(ax) for ax in (0, 1, 2)]
    return np.ascontiguousarray(arranged.transpose(perm))


# -- convolutions ----------------------------------------------------------------


def out_extent(n: int, f: int, s: int, p: int) -> int:
    """ConvGeometry.n_h / n_w (kernels.py:55-65)."""
    return (n + 2 * p - f) // s + 1


def sf_conv(x_chw_batch, nodes, seg_off, k_n, h_f, w_f, stride, pad, bias=None, threads=0):
    """Sparse-filter conv (layers.py:170-180 over kernels.py:78-97).

    x_chw_batch: (N, C, H, W) logical arrays.  nodes/seg_off: SparseTensor4 node
    buffer and global (K, H_F*W_F) segment table (CHW order).  Returns (N, K, n_h, n_w).
    """
    x = np.asarray(x_chw_batch, np.float32)
    n, c, h, w = x.shape
    whc = np.ascontiguousarray(x.transpose(0, 3, 2, 1))
    n_h, n_w = out_extent(h, h_f, stride, pad), out_extent(w, w_f, stride, pad)
    out = np.empty((n, n_w, n_h, k_n), np.float32)
    nodes = np.ascontiguousarray(nodes)
    seg = np.ascontiguousarray(seg_off, dtype=np.int64).ravel()
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    lib().oracle_sf_conv(_p(whc), n, c, h, w, _p(nodes), _p(seg), k_n, h_f, w_f, stride, pad,
                         None if b is None else _p(b), _p(out), int(threads))
    return np.ascontiguousarray(out.transpose(0, 3, 2, 1))


def sf_count(h_i, w_i, seg_off, n_nodes, k_n, h_f, w_f, stride, pad) -> int:
    """Exact multiply count of kernels.py:108-133 summed over the filter bank."""
    seg = np.ascontiguousarray(seg_off, dtype=np.int64).ravel()
    return int(lib().oracle_sf_count(h_i, w_i, _p(seg), n_nodes, k_n, h_f, w_f, stride, pad))


def si_conv(in_nodes_list, in_seg_list, dims_chw, filters_kchw, stride, pad, threads=0):
    """Sparse-input conv (kernels.py:136-166) for a batch of CHW node tensors.

    Returns dense (N, K, n_h, n_w) holding +0.0 wherever the reference stores no node.
    """
    c, h, w = dims_chw
    f = np.asarray(filters_kchw, np.float32)
    k_n, _, h_f, w_f = f.shape
    filt_whc = np.ascontiguousarray(f.transpose(0, 3, 2, 1))  # (K, W_F, H_F, C)
    bases = np.cumsum([0] + [len(x) for x in in_nodes_list[:-1]]).astype(np.int64)
    nodes = np.ascontiguousarray(np.concatenate(in_nodes_list))
    segs = np.ascontiguousarray(np.stack([np.asarray(s, np.int64) for s in in_seg_list]))
    n = len(in_nodes_list)
    n_h, n_w = out_extent(h, h_f, stride, pad), out_extent(w, w_f, stride, pad)
    out = np.empty((n, k_n, n_h, n_w), np.float32)
    lib().oracle_si_conv(_p(nodes), _p(bases), _p(segs), n, c, h, w, _p(filt_whc), k_n, h_f, w_f,
                         stride, pad, _p(out), int(threads))
    return out


def dense_conv(x_chw, filters_kchw, stride, pad, threads=0):
    """Dense oracle conv (kernels.py:169-192), (k, l, c) order.  Returns (K, n_h, n_w)."""
    x = np.asarray(x_chw, np.float32)
    c, h, w = x.shape
    whc = np.ascontiguousarray(x.transpose(2, 1, 0))
    f = np.asarray(filters_kchw, np.float32)
    k_n, _, h_f, w_f = f.shape
    filt_whc = np.ascontiguousarray(f.transpose(0, 3, 2, 1))
    n_h, n_w = out_extent(h, h_f, stride, pad), out_extent(w, w_f, stride, pad)
    out = np.empty((k_n, n_h, n_w), np.float32)
    lib().oracle_dense_conv(_p(whc), c, h, w, _p(filt_whc), k_n, h_f, w_f, stride, pad, _p(out),
                            int(threads))
    return out


def pool(x_chw_batch, h_p, w_p, mode="max"):
    """Dense pooling (layers.py:250-271).  (N, C, H, W) -> (N, C, H/h_p, W/w_p)."""
    x = np.asarray(x_chw_batch, np.float32)
    n, c, h, w = x.shape
    whc = np.ascontiguousarray(x.transpose(0, 3, 2, 1))
    out = np.empty((n, w // w_p, h // h_p, c), np.float32)
    lib().oracle_pool(_p(whc), n, c, h, w, h_p, w_p, 1 if mode == "max" else 0, _p(out))
    return np.ascontiguousarray(out.transpose(0, 3, 2, 1))


def relu(x):
    """np.maximum(x, 0) semantics (layers.py:482-483)."""
    a = np.ascontiguousarray(x, np.float32)
    out = np.empty_like(a)
    lib().oracle_relu(_p(a), a.size, _p(out))
    return out


# -- VGG16 conv stack ------------------------------------------------------------

VGG16_PLAN = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]


def encode_bank(filters_kchw: np.ndarray):
    """network.prepare's per-layer encoding (network.py:371-377): each filter
    sparsified in CHW order, then stacked.  Returns (nodes, seg_off[K, H_F*W_F])."""
    nodes, _, _, seg = encode_batch(filters_kchw, "CHW")
    return nodes, seg


def vgg_forward(x_nchw, banks, threads=0):
    """Sparse-filter VGG16 stack forward (network.py:410-461 path for vgg16_desk):
    conv (strategy II arithmetic) -> ReLU -> [2x2 max-pool after each block].

    banks: list of (nodes, seg_off, K, bias) per conv layer in plan order.
    Returns the final (N, 512, H/32, W/32) activations.
    """
    x = np.asarray(x_nchw, np.float32)
    li = 0
    for item in VGG16_PLAN:
        if item == "M":
            x = pool(x, 2, 2, "max")
        else:
            nodes, seg, k_n, bias = banks[li]
            x = relu(sf_conv(x, nodes, seg, k_n, 3, 3, 1, 1, bias, threads))
            li += 1
    return x


# -- sparse-input pipeline and node restructuring ------------------


def rebuild(nodes, seg_off, kind: str, slope: float = 0.0):
    """Node-format ReLU / LeakyReLU (layers.py:485-491 over sparse_core.py:460-473).
    Returns (nodes, seg_off) of the rebuilt tensor (same order and dims)."""
    nodes = np.ascontiguousarray(nodes)
    seg = np.ascontiguousarray(seg_off, dtype=np.int64)
    k = 0 if kind == "relu" else 1
    new_off = np.empty(seg.size, np.int64)
    L = lib()
    total = L.oracle_rebuild(_p(nodes), _p(seg), seg.size, k, float(np.float32(slope)), _p(new_off), None)
    out = np.empty(total, NODE_DTYPE)
    L.oracle_rebuild(_p(nodes), _p(seg), seg.size, k, float(np.float32(slope)), _p(new_off), _p(out))
    return out, new_off


def batchnorm(x_chw, scale, shift, mean, var, eps):
    """apply_batchnorm (layers.py:507-509) on a (C, H, W) array."""
    x = np.asarray(x_chw, np.float32)
    c, h, w = x.shape
    whc = np.ascontiguousarray(x.transpose(2, 1, 0))
    out = np.empty_like(whc)
    f = lambda a: np.ascontiguousarray(a, np.float32)
    sc, sh, mu, va = f(scale), f(shift), f(mean), f(var)
    lib().oracle_batchnorm(_p(whc), c, h * w, _p(sc), _p(sh), _p(mu), _p(va), float(np.float32(eps)), _p(out))
    return np.ascontiguousarray(out.transpose(2, 1, 0))


def pad_dense(x_chw, p: int):
    """pad_tensor on a dense (C, H, W) array (layers.py:518-520)."""
    x = np.asarray(x_chw, np.float32)
    c, h, w = x.shape
    whc = np.ascontiguousarray(x.transpose(2, 1, 0))
    out = np.empty((w + 2 * p, h + 2 * p, c), np.float32)
    lib().oracle_pad_dense(_p(whc), c, h, w, p, _p(out))
    return np.ascontiguousarray(out.transpose(2, 1, 0))


def pad_chw_nodes(nodes, seg_off, dims_chw, p: int):
    """pad_tensor on CHW nodes (layers.py:521-535): (nodes, seg_off) of the padded tensor."""
    c, h, w = dims_chw
    nodes = np.ascontiguousarray(nodes)
    seg = np.ascontiguousarray(seg_off, dtype=np.int64)
    new_off = np.empty((w + 2 * p) * (h + 2 * p), np.int64)
    L = lib()
    total = L.oracle_pad_chw_nodes(_p(nodes), _p(seg), h, w, p, _p(new_off), None)
    out = np.empty(total, NODE_DTYPE)
    L.oracle_pad_chw_nodes(_p(nodes), _p(seg), h, w, p, _p(new_off), _p(out))
    return out, new_off


def transpose_segments(nodes, seg_len: int):
    """transpose_matrix's re-bucketing (kernels.py:195-223, :360-380): (nodes, seg_off)."""
    nodes = np.ascontiguousarray(nodes)
    data = int((nodes["index"] != -1).sum())
    out = np.empty(data + seg_len, NODE_DTYPE)
    new_off = np.empty(seg_len, np.int64)
    cursor = np.empty(seg_len, np.int64)
    lib().oracle_transpose_segments(_p(nodes), len(nodes), seg_len, _p(new_off), _p(out), _p(cursor))
    return out, new_off


def transpose_whc_to_chw(nodes, seg_off, dims_chw):
    """transpose_tensor3 (kernels.py:383-411): WHC nodes -> CHW (nodes, seg_off)."""
    c, h, w = dims_chw
    nodes = np.ascontiguousarray(nodes)
    seg = np.ascontiguousarray(seg_off, dtype=np.int64)
    data = int((nodes["index"] != -1).sum())
    out = np.empty(data + w * h, NODE_DTYPE)
    new_off = np.empty(w * h, np.int64)
    cursor = np.empty(w * h, np.int64)
    lib().oracle_transpose_whc_to_chw(_p(nodes), _p(seg), c, h, w, _p(new_off), _p(out), _p(cursor))
    return out, new_off
