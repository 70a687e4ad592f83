"""Layer operators -- drop-in for the hot-path subset of sparse_infer.layers.

Strategy I (per-filter, layers.py:282-299) and strategy II (fused loop nest,
layers.py:302-323) are the same GPU launch here: all filters of the layer in one
kernel.  Their results are therefore bit-identical, as the reference guarantees, and
independent of ``workers`` (accepted for API compatibility; layers.py:149-155).

Kernel choice: 3x3 / stride 1 / pad 1 layers use the fast channel-major kernel
(fp32 reassociation, held to 1e-4 normwise); any other geometry -- or
``set_exact(True)`` / FSCNN_EXACT=1 -- uses the reference-order kernel, bit-exact with
the reference.
"""

from __future__ import annotations

import os
from dataclasses import dataclass
from enum import Enum

import numpy as np

from . import kernels
from .kernels import ConvGeometry
from .sparse_core import (
    AxisOrder2,
    AxisOrder3,
    DenseTensor3,
    SparseMatrix,
    SparseTensor3,
    SparseTensor4,
)

POOL_MAX = "max"
POOL_AVG = "avg"

_EXACT = os.environ.get("FSCNN_EXACT", "0") == "1"


def set_exact(flag: bool) -> None:
    """Force the reference-order (bit-exact) sparse-filter kernel for every geometry."""
    global _EXACT
    _EXACT = bool(flag)


@dataclass(frozen=True)
class LayerSpec:
    """One layer of a sequential stack (layers.py:46-79)."""

    kind: str
    out_channels: int = 0
    kernel: tuple[int, int] = (0, 0)
    stride: int = 1
    padding: int = 0
    slope: float = 0.0

    def out_dims(self, in_dims):
        c, h, w = in_dims
        if self.kind == "conv":
            g = ConvGeometry(in_dims, (c,) + tuple(self.kernel), self.stride, self.padding)
            return (self.out_channels, g.n_h, g.n_w)
        if self.kind in ("maxpool", "avgpool"):
            h_p, w_p = self.kernel
            if h_p <= 0 or w_p <= 0:
                raise ValueError(f"pool window must be positive, got {self.kernel}")
            if h % h_p or w % w_p:
                raise ValueError(f"input {h}x{w} not divisible by pool window {h_p}x{w_p}")
            return (c, h // h_p, w // w_p)
        if self.kind == "pad":
            return (c, h + 2 * self.padding, w + 2 * self.padding)
        if self.kind in ("relu", "leaky_relu", "batchnorm"):
            return tuple(in_dims)
        raise ValueError(f"unknown layer kind {self.kind!r}")


class StrategyKind(Enum):
    STRATEGY_I = "1"
    STRATEGY_II = "2"
    AUTO = "auto"


@dataclass(frozen=True)
class ForwardStrategy:
    """Auto switch on batch size, threshold 4 (layers.py:88-104)."""

    kind: StrategyKind = StrategyKind.AUTO
    threshold: int = 4

    def __post_init__(self):
        if self.threshold < 1:
            raise ValueError("auto-switch threshold must be positive")

    def resolve(self, batch_size: int) -> StrategyKind:
        if self.kind is not StrategyKind.AUTO:
            return self.kind
        return StrategyKind.STRATEGY_I if batch_size <= self.threshold else StrategyKind.STRATEGY_II


# -- sparse-filter conv layer ---------------------------------------------------------

_bank_cache: dict = {}


def _device_bank(filters: SparseTensor4):
    """Device copies of a host SparseTensor4 (+ its fast-kernel pack), cached per object."""
    import torch

    from . import device

    key = id(filters)
    hit = _bank_cache.get(key)
    if hit is not None and hit[0] is filters:
        return hit[1]
    k, c, h_f, w_f = filters.dims
    nodes = device.nodes_from_numpy(filters.nodes)
    seg = torch.from_numpy(np.ascontiguousarray(filters.segment_offsets, dtype=np.int64).ravel()).cuda()
    packed = None
    if (h_f, w_f) == (3, 3):
        dense = torch.empty((k, c, 3, 3), dtype=torch.float32, device="cuda")
        # segment (k, w*3 + h) holds channel fiber c -> dense[k][c][h][w]
        device.decode(nodes, seg, k, 3, 3, c, dense, (c * 9, 1, 3, 9))
        packed = device.sf_pack(dense)
    entry = (nodes, seg, packed)
    if len(_bank_cache) > 64:
        _bank_cache.clear()
    _bank_cache[key] = (filters, entry)
    return entry


def _sf_layer(t_in: DenseTensor3, filters: SparseTensor4, stride: int, padding: int, bias) -> DenseTensor3:
    import torch

    from . import device

    if filters.order is not AxisOrder3.CHW:
        raise ValueError(f"filters must be stored CHW, got {filters.order.name}")
    geom = ConvGeometry(tuple(t_in.dims), tuple(filters.dims[1:]), stride, padding)
    k = filters.count
    nodes, seg, packed = _device_bank(filters)
    b = torch.from_numpy(np.ascontiguousarray(bias, dtype=np.float32)).cuda()
    x = kernels.dense_to_device(t_in)
    if packed is not None and stride == 1 and padding == 1 and not _EXACT:
        c, h, w = t_in.dims
        y = device.sf_conv3x3(device.to_halo(x), packed, b, relu=False, pool=False, w=w)
        y = device.from_halo(y, w).contiguous()
    else:
        _, h_f, w_f = filters.dims[1:]
        y = device.sf_conv_exact(x, nodes, seg, k, h_f, w_f, stride, padding, b)
    return kernels.dense_from_device(y)


def conv_forward_strategy_I(t_in: DenseTensor3, filters: SparseTensor4, stride: int, padding: int,
                            bias: np.ndarray, workers: int = 1) -> DenseTensor3:
    """Per-filter strategy (layers.py:282-299); same GPU launch as strategy II."""
    return _sf_layer(t_in, filters, stride, padding, bias)


def conv_forward_strategy_II(t_in: DenseTensor3, filters: SparseTensor4, stride: int, padding: int,
                             bias: np.ndarray) -> DenseTensor3:
    """Fused strategy (layers.py:302-323)."""
    return _sf_layer(t_in, filters, stride, padding, bias)


# -- sparse-input conv layer ----------------------------------------------------------


def _si_dense(t_in: SparseTensor3, filters: list[DenseTensor3], stride: int, padding: int):
    from . import device

    if t_in.order is not AxisOrder3.CHW:
        raise ValueError(f"input tensor must be stored CHW, got {t_in.order.name}")
    geom = ConvGeometry(tuple(t_in.dims), tuple(filters[0].dims), stride, padding)
    nodes, seg = kernels.sparse_to_device(t_in)
    c, h, w = t_in.dims
    _, h_f, w_f = filters[0].dims
    kcrs = kernels.filters_to_device_kcrs(filters)
    if (h_f, w_f, stride, padding) == (3, 3, 1, 1):
        y = device.si_conv3x3(nodes, seg, 1, c, h, w, device.si_pack3x3(kcrs), len(filters))
    else:
        y = device.si_conv(nodes, seg, 1, c, h, w, device.kcrs_to_crsk(kcrs), len(filters), h_f, w_f, stride, padding)
    return y, geom


def _pool_args(pool, mode, n_h, n_w):
    h_p, w_p = pool
    if h_p <= 0 or w_p <= 0:
        raise ValueError(f"pool window must be positive, got {pool}")
    if n_h % h_p or n_w % w_p:
        raise ValueError(f"conv output {n_h}x{n_w} not divisible by pool {h_p}x{w_p}")
    if mode not in (POOL_MAX, POOL_AVG):
        raise ValueError(f"unknown pool mode {mode!r}")
    return h_p, w_p


def conv_forward_sparse_input(t_in: SparseTensor3, filters: list[DenseTensor3], stride: int, padding: int,
                              bias: np.ndarray, workers: int = 1, fused_pool=None, pool_mode: str = POOL_MAX):
    """Sparse-input layer (layers.py:393-429): CHW node output when bias == 0, else a
    DenseTensor3.  A fused pool (Alg. 7) equals conv followed by pooling exactly
    (layers.py:345-390), which is how it runs here."""
    import torch

    from . import device

    y, geom = _si_dense(t_in, filters, stride, padding)
    if fused_pool is not None:
        h_p, w_p = _pool_args(fused_pool, pool_mode, geom.n_h, geom.n_w)
        y = device.pool2d(y, h_p, w_p, pool_mode == POOL_MAX)
    bias = np.asarray(bias, dtype=np.float32)
    if np.any(bias != 0):
        y = y + torch.from_numpy(bias).cuda().view(1, -1, 1, 1)
        return kernels.dense_from_device(y)
    enc = device.encode_order(y, "CHW")
    k, n_h, n_w = (int(v) for v in y.shape[1:])
    return SparseTensor3(AxisOrder3.CHW, (k, n_h, n_w), device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                         enc.matrix_off.cpu().numpy(), enc.seg_off.cpu().numpy())


def merged_conv_pool(t_in: SparseTensor3, t_f: DenseTensor3, stride: int, pool, mode: str,
                     padding: int = 0) -> SparseMatrix:
    """Alg. 7 conv+pool for one filter (layers.py:345-390) -> WH SparseMatrix."""
    from . import device

    geom = ConvGeometry(tuple(t_in.dims), tuple(t_f.dims), stride, padding)
    h_p, w_p = _pool_args(pool, mode, geom.n_h, geom.n_w)
    y, _ = _si_dense(t_in, [t_f], stride, padding)
    y = device.pool2d(y, h_p, w_p, mode == POOL_MAX)
    n_h, n_w = geom.n_h // h_p, geom.n_w // w_p
    enc = device.encode(y, 1, 1, n_h, n_w, (0, 0, n_w, 1))
    return SparseMatrix(AxisOrder2.WH, n_h, n_w, device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                        enc.seg_off.cpu().numpy())


# -- dense layers between convolutions ---------------------------------------------------


def pool_standalone(t: DenseTensor3, pool, mode: str) -> DenseTensor3:
    """Non-overlapping window pooling (layers.py:449-461) on the GPU."""
    from . import device

    c, h, w = t.dims
    h_p, w_p = pool
    if h_p <= 0 or w_p <= 0:
        raise ValueError(f"pool window must be positive, got {pool}")
    if h % h_p or w % w_p:
        raise ValueError(f"input {h}x{w} not divisible by pool window {h_p}x{w_p}")
    if mode not in (POOL_MAX, POOL_AVG):
        raise ValueError(f"unknown pool mode {mode!r}")
    y = device.pool2d(kernels.dense_to_device(t), h_p, w_p, mode == POOL_MAX)
    return kernels.dense_from_device(y)


def apply_activation(t, kind: str, slope: float = 0.0):
    """ReLU on dense tensors (layers.py:469-484) on the GPU.

    LeakyReLU and node-format activations belong to the sparse-input pipeline
    (not built yet) and raise NotImplementedError.
    """
    if kind not in ("relu", "leaky_relu"):
        raise ValueError(f"unknown activation {kind!r}")
    if slope < 0:
        raise ValueError("leaky slope must be non-negative")
    if isinstance(t, DenseTensor3) and kind == "relu":
        import torch

        from . import device

        flat = torch.from_numpy(np.ascontiguousarray(t.data)).cuda()
        return DenseTensor3(tuple(t.dims), device.relu(flat).cpu().numpy())
    if isinstance(t, (DenseTensor3, SparseTensor3)):
        raise NotImplementedError(f"{kind} on {type(t).__name__} is outside the built hot path (SURVEY.md §8f-1)")
    raise TypeError(f"apply_activation does not support {type(t).__name__}")
