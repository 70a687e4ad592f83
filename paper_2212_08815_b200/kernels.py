"""Convolution operators -- drop-in for sparse_infer.kernels.

``conv_dense_input_sparse_filter[_counted]`` (kernels.py:264-305),
``conv_sparse_input_dense_filter`` (kernels.py:308-339), ``dense_conv_reference``
(:342-350), ``dot_dense_sparse`` (:352-358) and the node-format transposes
``transpose_matrix`` / ``transpose_tensor3`` (:360-411) keep the reference's
signatures, validation and error messages; the arithmetic runs on the GPU in the
reference's accumulation order (bit-exact; see fscnn_sf_conv_exact / fscnn_si_conv /
fscnn_dense_conv_exact), and the transposes move nodes without touching values.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .sparse_core import (
    AxisOrder2,
    AxisOrder3,
    DenseTensor3,
    FormatError,
    SparseMatrix,
    SparseTensor3,
    SparseVector,
)


@dataclass(frozen=True)
class ConvGeometry:
    """Shape contract of one convolution (kernels.py:34-65)."""

    input_dims: tuple[int, int, int]
    filter_dims: tuple[int, int, int]
    stride: int = 1
    padding: int = 0

    def __post_init__(self):
        c_i, h_i, w_i = self.input_dims
        c_f, h_f, w_f = self.filter_dims
        if self.stride <= 0:
            raise ValueError(f"stride must be positive, got {self.stride}")
        if self.padding < 0:
            raise ValueError(f"padding must be non-negative, got {self.padding}")
        if c_i != c_f:
            raise ValueError(f"channel mismatch: input C={c_i}, filter C={c_f}")
        if h_f > h_i + 2 * self.padding or w_f > w_i + 2 * self.padding:
            raise ValueError(f"filter {self.filter_dims} exceeds padded input {self.input_dims}")

    @property
    def n_h(self) -> int:
        return (self.input_dims[1] + 2 * self.padding - self.filter_dims[1]) // self.stride + 1

    @property
    def n_w(self) -> int:
        return (self.input_dims[2] + 2 * self.padding - self.filter_dims[2]) // self.stride + 1


def _require_order3(t: SparseTensor3, order: AxisOrder3, what: str) -> None:
    if t.order is not order:
        raise FormatError(f"{what} must be stored {order.name}, got {t.order.name}")


def _check_conv_args(input_dims, filter_dims, geom: ConvGeometry) -> None:
    if tuple(input_dims) != tuple(geom.input_dims):
        raise ValueError(f"input dims {input_dims} != geometry {geom.input_dims}")
    if tuple(filter_dims) != tuple(geom.filter_dims):
        raise ValueError(f"filter dims {filter_dims} != geometry {geom.filter_dims}")


# -- device staging helpers ----------------------------------------------------------


def _torch():
    from . import _lib

    _lib.require_cuda()
    import torch

    return torch


def dense_to_device(t: DenseTensor3):
    """Host DenseTensor3 (W,H,C memory) -> device NCHW [1, C, H, W] (GPU transpose); a
    DeviceDenseTensor3 is already that tensor."""
    from .sparse_core import DeviceDenseTensor3

    if isinstance(t, DeviceDenseTensor3):
        t.validate()
        return t.data
    torch = _torch()
    from . import device

    c, h, w = t.dims
    flat = torch.from_numpy(np.ascontiguousarray(t.data)).cuda()
    return device.whc_to_nchw(flat, 1, c, h, w)


def dense_from_device(y, resident: bool = False) -> DenseTensor3:
    """Device [1, K, H, W] -> host DenseTensor3 (GPU transpose to W,H,C, then D2H), or
    (resident) a DeviceDenseTensor3 around it."""
    from . import device

    if resident:
        from .sparse_core import DeviceDenseTensor3

        y = y.contiguous()
        return DeviceDenseTensor3(tuple(int(v) for v in y.shape[1:]), y)

    _, k, h, w = (int(v) for v in y.shape)
    whc = device.nchw_to_whc(y)
    return DenseTensor3((k, h, w), whc.cpu().numpy().ravel())


def sparse_to_device(t: SparseTensor3):
    """Host SparseTensor3 -> (device nodes, device segment offsets).  The structure is
    validated first (sorted in-range indices, sentinel-terminated segments): the kernels
    trust it, and a malformed fiber would index shared memory out of bounds."""
    from .sparse_core import DeviceSparseTensor3

    if isinstance(t, DeviceSparseTensor3):
        t.validate()
        return t.nodes, t.segment_offsets
    torch = _torch()
    from . import device

    t.validate()

    return (device.nodes_from_numpy(t.nodes),
            torch.from_numpy(np.ascontiguousarray(t.segment_offsets, dtype=np.int64)).cuda())


def filters_to_device_kcrs(filters: list[DenseTensor3]):
    """list of K (C, H_F, W_F) DenseTensor3 -> device dense [K, C, H_F, W_F]."""
    torch = _torch()
    c, h_f, w_f = filters[0].dims
    stacked = np.stack([np.asarray(f.data, np.float32) for f in filters])  # (K, W_F*H_F*C)
    dev = torch.from_numpy(stacked).cuda().view(len(filters), w_f, h_f, c)
    return dev.permute(0, 3, 2, 1).contiguous()


# -- operators -----------------------------------------------------------------------


def _sf_single(t_in: DenseTensor3, t_f: SparseTensor3, geom: ConvGeometry) -> np.ndarray:
    from . import device

    x = dense_to_device(t_in)
    nodes, seg = sparse_to_device(t_f)
    c_f, h_f, w_f = t_f.dims
    y = device.sf_conv_exact(x, nodes, seg, 1, h_f, w_f, geom.stride, geom.padding, None)
    return y[0, 0].cpu().numpy()


def conv_dense_input_sparse_filter(t_in: DenseTensor3, t_f: SparseTensor3, geom: ConvGeometry) -> np.ndarray:
    """Dense input x one CHW sparse filter -> dense (n_h, n_w) (kernels.py:264-283)."""
    _require_order3(t_f, AxisOrder3.CHW, "filter tensor")
    _check_conv_args(t_in.dims, t_f.dims, geom)
    return _sf_single(t_in, t_f, geom)


def multiply_count(t_f: SparseTensor3, geom: ConvGeometry) -> int:
    """Exact in-bounds multiply tally of the counted kernel (kernels.py:108-133):
    sum over taps of nnz(tap segment) x valid output rows x valid output columns."""
    c_f, h_f, w_f = t_f.dims
    h_i, w_i = geom.input_dims[1], geom.input_dims[2]
    s, p = geom.stride, geom.padding
    seg = np.asarray(t_f.segment_offsets, np.int64)
    ends = np.append(seg[1:], len(t_f.nodes))
    nnz = ends - seg - 1
    total = 0
    for tap in range(h_f * w_f):
        l, k = divmod(tap, h_f)
        rows = sum(1 for i in range(geom.n_h) if 0 <= k + i * s - p < h_i)
        cols = sum(1 for j in range(geom.n_w) if 0 <= l + j * s - p < w_i)
        total += int(nnz[tap]) * rows * cols
    return total


def conv_dense_input_sparse_filter_counted(t_in: DenseTensor3, t_f: SparseTensor3, geom: ConvGeometry):
    """Same result plus the exact multiply count (kernels.py:286-305)."""
    _require_order3(t_f, AxisOrder3.CHW, "filter tensor")
    _check_conv_args(t_in.dims, t_f.dims, geom)
    return _sf_single(t_in, t_f, geom), multiply_count(t_f, geom)


def conv_sparse_input_dense_filter(t_in: SparseTensor3, t_f: DenseTensor3, geom: ConvGeometry) -> SparseMatrix:
    """CHW sparse input x one dense filter -> WH SparseMatrix of the nonzero outputs
    (kernels.py:308-339): the GPU computes the dense plane in the reference's order and
    the GPU encoder keeps exactly the entries that compare != 0."""
    _require_order3(t_in, AxisOrder3.CHW, "input tensor")
    _check_conv_args(t_in.dims, t_f.dims, geom)
    from . import device

    nodes, seg = sparse_to_device(t_in)
    c, h, w = t_in.dims
    _, h_f, w_f = t_f.dims
    wt = device.kcrs_to_crsk(filters_to_device_kcrs([t_f]))
    y = device.si_conv(nodes, seg, 1, c, h, w, wt, 1, h_f, w_f, geom.stride, geom.padding)
    enc = device.encode(y, 1, 1, geom.n_h, geom.n_w, (0, 0, geom.n_w, 1))
    return SparseMatrix(AxisOrder2.WH, geom.n_h, geom.n_w, device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                        enc.seg_off.cpu().numpy())


def dense_conv_reference(t_in: DenseTensor3, t_f: DenseTensor3, geom: ConvGeometry) -> np.ndarray:
    """Dense cross-correlation with one filter (kernels.py:342-350): the GPU dense kernel
    in _dense_conv_kernel's (kh, kw, c) order, bit-exact."""
    _check_conv_args(t_in.dims, t_f.dims, geom)
    from . import device

    y = device.dense_conv_exact(dense_to_device(t_in), filters_to_device_kcrs([t_f]), geom.stride,
                                geom.padding, None)
    return y[0, 0].cpu().numpy()


def dot_dense_sparse(d: np.ndarray, s: SparseVector) -> float:
    """Inner product of a dense fiber with a sparse vector in node order (kernels.py:352-358):
    the reference-order sparse-filter kernel on a 1x1 "image" of len(d) channels."""
    d = np.ascontiguousarray(d, dtype=np.float32)
    s.validate()
    if s.length > len(d):
        raise FormatError(f"sparse length {s.length} exceeds dense length {len(d)}")
    torch = _torch()
    from . import device

    x = torch.from_numpy(d).cuda().view(1, len(d), 1, 1)
    nodes = device.nodes_from_numpy(s.nodes)
    seg = torch.zeros(1, dtype=torch.int64, device="cuda")
    return float(device.sf_conv_exact(x, nodes, seg, 1, 1, 1, 1, 0, None)[0, 0, 0, 0].item())


def transpose_matrix(m: SparseMatrix) -> SparseMatrix:
    """WH <-> HW storage switch (kernels.py:360-380) on the GPU: decode with a presence
    mask, masked re-encode in the other order -- every stored node (explicit zeros
    too) moves with its value untouched."""
    torch = _torch()
    from . import device

    dense = torch.zeros((m.n_rows, m.n_cols), dtype=torch.float32, device="cuda")
    mask = torch.zeros((m.n_rows, m.n_cols), dtype=torch.uint8, device="cuda")
    row_major = (0, 0, m.n_cols, 1)   # WH: segment = row, index = column
    col_major = (0, 0, 1, m.n_cols)   # HW: segment = column, index = row
    src, dst = (row_major, col_major) if m.order is AxisOrder2.WH else (col_major, row_major)
    if m.n_segments and m.segment_length:
        device.decode(device.nodes_from_numpy(m.nodes), torch.from_numpy(np.asarray(m.segment_offsets, np.int64)).cuda(),
                      1, 1, m.n_segments, m.segment_length, dense, src, mask)
    flipped = AxisOrder2.HW if m.order is AxisOrder2.WH else AxisOrder2.WH
    n_seg, seg_len = (m.n_cols, m.n_rows) if flipped is AxisOrder2.HW else (m.n_rows, m.n_cols)
    enc = device.encode(dense, 1, 1, n_seg, seg_len, dst, mask=mask)
    return SparseMatrix(flipped, m.n_rows, m.n_cols, device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                        enc.seg_off.cpu().numpy())


def transpose_tensor3(t: SparseTensor3) -> SparseTensor3:
    """WHC -> CHW without touching any value (kernels.py:383-411), on the GPU: masked
    decode from WHC, masked encode in CHW."""
    _require_order3(t, AxisOrder3.WHC, "tensor")
    torch = _torch()
    from . import device

    c, h, w = t.dims
    dense = torch.zeros((1, c, h, w), dtype=torch.float32, device="cuda")
    mask = torch.zeros((1, c, h, w), dtype=torch.uint8, device="cuda")
    if t.n_segments:
        device.decode_order(device.nodes_from_numpy(t.nodes), torch.from_numpy(np.asarray(t.segment_offsets, np.int64)).cuda(),
                            (1, c, h, w), "WHC", out=dense, mask=mask)
    enc = device.encode_order(dense, "CHW", mask=mask)
    return SparseTensor3(AxisOrder3.CHW, tuple(t.dims), device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                         enc.matrix_off.cpu().numpy(), enc.seg_off.cpu().numpy())
