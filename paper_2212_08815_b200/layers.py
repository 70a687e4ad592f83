"""Layer operators -- drop-in for the hot-path subset of sparse_infer.layers.

Strategy I (per-filter, layers.py:282-299) and strategy II (fused loop nest,
layers.py:302-323) are the same GPU launch here: all filters of the layer in one
kernel.  Their results are therefore bit-identical, as the reference guarantees, and
independent of ``workers`` (accepted for API compatibility; layers.py:149-155).

Kernel choice: 3x3 / stride 1 / pad 1 layers big enough to fill the GPU use the fast
channel-major kernels (fp32 reassociation, held to 1e-4 normwise; sparse-filter and
sparse-input alike); smaller ones (one 56x56 image, as config 1; config 2), any other
geometry, or ``set_exact(True)`` / FSCNN_EXACT=1 use the reference-order kernels,
bit-exact with the reference.
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
    DeviceDenseTensor3,
    DeviceSparseTensor3,
    SparseMatrix,
    SparseTensor3,
    SparseTensor4,
    _sparse_result,
)

POOL_MAX = "max"
POOL_AVG = "avg"

_DENSE = (DenseTensor3, DeviceDenseTensor3)
_SPARSE = (SparseTensor3, DeviceSparseTensor3)


def _resident(t) -> bool:
    """A device twin in means a device twin out (the chain stays on the GPU)."""
    return isinstance(t, (DeviceDenseTensor3, DeviceSparseTensor3))

_EXACT = os.environ.get("FSCNN_EXACT", "0") == "1"


def set_exact(flag: bool) -> None:
    """Force the reference-order (bit-exact) sparse-filter and sparse-input kernels for
    every geometry."""
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


_LAYER_JIT = os.environ.get("FSCNN_LAYER_JIT", "1") != "0"
_jit_cache: dict = {}


def _layer_jit(filters: SparseTensor4, bias, h: int, w: int):
    """The single-kernel specialised conv of a bank (+ bias, no ReLU/pool), cached."""
    import torch

    from . import device

    b = np.ascontiguousarray(bias, dtype=np.float32)
    key = (id(filters), b.tobytes(), h, w)
    hit = _jit_cache.get(key)
    if hit is not None and hit[0] is filters:
        return hit[1]
    nodes, seg, _ = _device_bank(filters)
    k, c = filters.dims[:2]
    dense = torch.empty((k, c, 3, 3), dtype=torch.float32, device="cuda")
    device.decode(nodes, seg, k, 3, 3, c, dense, (c * 9, 1, 3, 9))
    jit = device.SfJit(dense, b, h, w, relu=False, pool=False, flags=4 | (8 << 8) | (1 << 16))
    if len(_jit_cache) > 32:
        _jit_cache.clear()
    _jit_cache[key] = (filters, jit)
    return jit


def _small_bank(filters: SparseTensor4, kt: int):
    """The fast kernel's packed stream with ``kt`` filters per warp (cached with the bank)."""
    import torch

    from . import device

    hit = _bank_cache.get(("small", id(filters), kt))
    if hit is not None and hit[0] is filters:
        return hit[1]
    nodes, seg, _ = _device_bank(filters)
    k, c = filters.dims[:2]
    dense = torch.empty((k, c, 3, 3), dtype=torch.float32, device="cuda")
    device.decode(nodes, seg, k, 3, 3, c, dense, (c * 9, 1, 3, 9))
    bank = device.sf_pack(dense, kt)
    _bank_cache[("small", id(filters), kt)] = (filters, bank)
    return bank


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
    c, h, w = t_in.dims
    if packed is not None and stride == 1 and padding == 1 and not _EXACT and h % 2 == 0 and w % 2 == 0 \
            and device.sfjit_enabled() and _LAYER_JIT:
        # one layer call = one image: the bank compiled into ONE specialised kernel
        # (4 filters per group, blockIdx.y = group, 8-warp CTAs) -- config 1: 3.8 us
        # graph-launched vs 11.9 for the jump-table kernel's small-grid plan and 13.2 for
        # the reference-order kernel (profiles/r02_configs_12.json); bit-identical to
        # the jump-table kernel.  Compiled on first use, cached with the bank.
        jit = _layer_jit(filters, bias, h, w)
        y = device.from_halo(jit(device.to_halo(x)), w).contiguous()
        return kernels.dense_from_device(y, _resident(t_in))
    if packed is not None and stride == 1 and padding == 1 and not _EXACT:
        # the fast kernel, with its small-grid plan (fewer filters per warp, more CTAs)
        # when the default grid would leave SMs idle -- one image of config 1: 11.9 us
        # vs 13.2 for the reference-order kernel (profiles/r02_configs_12.json)
        kt, warps = device.sf_grid_plan(1, h, w, k, device.pick_ly(c, h))
        bank = packed if kt == packed.kt else _small_bank(filters, kt)
        y = device.sf_conv3x3(device.to_halo(x), bank, b, relu=False, pool=False, w=w, cta_warps=warps)
        y = device.from_halo(y, w).contiguous()
    else:
        _, h_f, w_f = filters.dims[1:]
        y = device.sf_conv_exact(x, nodes, seg, k, h_f, w_f, stride, padding, b)
    return kernels.dense_from_device(y, _resident(t_in))


def conv_forward_strategy_I(t_in: DenseTensor3, filters: SparseTensor4, stride: int, padding: int,
                            bias: np.ndarray, workers: int = 1) -> DenseTensor3:
    """Per-filter strategy (layers.py:282-299); same GPU launch as strategy II."""
    return _sf_layer(t_in, filters, stride, padding, bias)


def conv_forward_strategy_II(t_in: DenseTensor3, filters: SparseTensor4, stride: int, padding: int,
                             bias: np.ndarray) -> DenseTensor3:
    """Fused strategy (layers.py:302-323)."""
    return _sf_layer(t_in, filters, stride, padding, bias)


# -- sparse-input conv layer ----------------------------------------------------------


def _si_dense(t_in: SparseTensor3, filters: list[DenseTensor3], stride: int, padding: int,
              fused_pool=None, pool_mode: str = POOL_MAX):
    """The conv on the device; with a 2x2 ``fused_pool`` on the channel-major path the
    pool runs in the kernel's epilogue (Alg. 7) and the result is already pooled."""
    from . import device

    if t_in.order is not AxisOrder3.CHW:
        raise ValueError(f"input tensor must be stored CHW, got {t_in.order.name}")
    geom = ConvGeometry(tuple(t_in.dims), tuple(filters[0].dims), stride, padding)
    nodes, seg = kernels.sparse_to_device(t_in)
    c, h, w = t_in.dims
    _, h_f, w_f = filters[0].dims
    kcrs = kernels.filters_to_device_kcrs(filters)
    k = len(filters)
    if (h_f, w_f, stride, padding) == (3, 3, 1, 1) and not _EXACT and device.si_use_fast(h, w, k):
        fp = None
        if fused_pool is not None and tuple(fused_pool) == (2, 2) and h % 2 == 0 and w % 2 == 0 and \
                pool_mode in (POOL_MAX, POOL_AVG):
            fp = "max" if pool_mode == POOL_MAX else "avg"
        y = device.si_conv3x3_fast(nodes, seg, 1, c, h, w, device.si_pack_fast(kcrs), k, pool=fp)
    elif (h_f, w_f, stride, padding) == (3, 3, 1, 1):
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

    if fused_pool is not None:  # validate the window before any device work
        g0 = ConvGeometry(tuple(t_in.dims), tuple(filters[0].dims), stride, padding)
        _pool_args(fused_pool, pool_mode, g0.n_h, g0.n_w)
    y, geom = _si_dense(t_in, filters, stride, padding, fused_pool, pool_mode)
    if fused_pool is not None and tuple(y.shape[2:]) == (geom.n_h, geom.n_w):
        h_p, w_p = _pool_args(fused_pool, pool_mode, geom.n_h, geom.n_w)
        y = device.pool2d(y, h_p, w_p, pool_mode == POOL_MAX)
    bias = np.asarray(bias, dtype=np.float32)
    if np.any(bias != 0):
        y = y + torch.from_numpy(bias).cuda().view(1, -1, 1, 1)
        return kernels.dense_from_device(y, _resident(t_in))
    return _sparse_result(device.encode_order(y, "CHW"), AxisOrder3.CHW, y.shape[1:], _resident(t_in))


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
    return kernels.dense_from_device(y, _resident(t))


def pool_sparse(t: SparseTensor3, pool, mode: str) -> SparseTensor3:
    """Node-format pooling (layers.py:464-466): decode, pool, re-encode in t.order -- all
    on the GPU, no host round trip in between."""
    from . import device
    from .sparse_core import from_device_dense, to_device_dense

    c, h, w = t.dims
    h_p, w_p = pool
    if h_p <= 0 or w_p <= 0:
        raise ValueError(f"pool window must be positive, got {pool}")
    if h % h_p or w % w_p:
        raise ValueError(f"input {h}x{w} not divisible by pool window {h_p}x{w_p}")
    if mode not in (POOL_MAX, POOL_AVG):
        raise ValueError(f"unknown pool mode {mode!r}")
    y = device.pool2d(to_device_dense(t), h_p, w_p, mode == POOL_MAX)
    return from_device_dense(y, t.order, _resident(t))


def apply_activation(t, kind: str, slope: float = 0.0):
    """ReLU / LeakyReLU keeping the representation (layers.py:469-492), on the GPU.

    Dense: np.maximum(x, 0) / np.where(x > 0, x, s*x).  Node format: the reference's
    rebuild_tensor3 (sparse_core.py:460-473) -- ReLU keeps nodes with value > 0 (NaN and
    -0.0 dropped), LeakyReLU rescales negative nodes and keeps the nonzero results --
    done as decode -> elementwise -> re-encode, which yields the same nodes and offsets
    because a valid segment's indices ascend.
    """
    if kind not in ("relu", "leaky_relu"):
        raise ValueError(f"unknown activation {kind!r}")
    if slope < 0:
        raise ValueError("leaky slope must be non-negative")
    from . import device

    if isinstance(t, DeviceDenseTensor3):
        t.validate()
        y = device.activation(t.data, device.ACT_RELU if kind == "relu" else device.ACT_LEAKY, slope)
        return DeviceDenseTensor3(tuple(t.dims), y)
    if isinstance(t, DenseTensor3):
        flat = kernels._torch().from_numpy(np.ascontiguousarray(t.data)).cuda()
        y = device.activation(flat, device.ACT_RELU if kind == "relu" else device.ACT_LEAKY, slope)
        return DenseTensor3(tuple(t.dims), y.cpu().numpy())
    if isinstance(t, _SPARSE):
        from .sparse_core import from_device_dense, to_device_dense

        act = device.ACT_RELU_NODES if kind == "relu" else device.ACT_LEAKY
        return from_device_dense(device.activation(to_device_dense(t), act, slope), t.order, _resident(t))
    raise TypeError(f"apply_activation does not support {type(t).__name__}")


@dataclass(frozen=True)
class BatchNormParams:
    """Per-channel inference statistics, all float32 incl. epsilon (layers.py:108-133)."""

    scale: np.ndarray
    shift: np.ndarray
    mean: np.ndarray
    var: np.ndarray
    epsilon: float = 1e-5

    def __post_init__(self):
        for name in ("scale", "shift", "mean", "var"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), dtype=np.float32))
        object.__setattr__(self, "epsilon", float(np.float32(self.epsilon)))

    def validate(self, channels: int) -> None:
        for name in ("scale", "shift", "mean", "var"):
            if getattr(self, name).shape != (channels,):
                raise ValueError(f"batchnorm {name} must have shape ({channels},)")
        if np.any(self.var + np.float32(self.epsilon) <= 0):
            raise ValueError("batchnorm requires var + epsilon > 0 per channel")


def apply_batchnorm(t, params: BatchNormParams):
    """Inference batch norm (layers.py:495-510) on the GPU; node-format input is decoded,
    normalised and re-encoded in its order (the result is dense in general)."""
    from . import device

    params.validate(t.dims[0])
    if isinstance(t, _SPARSE):
        from .sparse_core import from_device_dense, to_device_dense

        y = device.batchnorm(to_device_dense(t), params.scale, params.shift, params.mean, params.var,
                             params.epsilon)
        return from_device_dense(y, t.order, _resident(t))
    if not isinstance(t, _DENSE):
        raise TypeError(f"apply_batchnorm does not support {type(t).__name__}")
    y = device.batchnorm(kernels.dense_to_device(t), params.scale, params.shift, params.mean, params.var,
                         params.epsilon)
    return kernels.dense_from_device(y, _resident(t))


def pad_tensor(t, p: int):
    """Zero-pad the spatial extents by p (layers.py:513-540).  CHW node tensors keep every
    node (explicit zeros too): only segment placement changes, a device segment gather."""
    if p < 0:
        raise ValueError("pad width must be non-negative")
    if p == 0:
        return t
    from . import device

    if isinstance(t, _DENSE):
        return kernels.dense_from_device(device.pad2d(kernels.dense_to_device(t), p), _resident(t))
    if isinstance(t, _SPARSE):
        from .sparse_core import from_device_dense, to_device_dense

        if t.order is not AxisOrder3.CHW:
            return from_device_dense(device.pad2d(to_device_dense(t), p), t.order, _resident(t))
        torch = kernels._torch()
        c, h, w = t.dims
        nh, nw = h + 2 * p, w + 2 * p
        # new segment w'*nh + h' <- old (w'-p)*h + (h'-p) inside, else empty
        wi = torch.arange(nw, device="cuda").view(nw, 1) - p
        hi = torch.arange(nh, device="cuda").view(1, nh) - p
        inside = (wi >= 0) & (wi < w) & (hi >= 0) & (hi < h)
        seg_map = torch.where(inside, wi * h + hi, torch.full_like(wi * hi, -1)).view(-1)
        nodes, seg = kernels.sparse_to_device(t)
        out, count, off = device.remap_segments(nodes, seg, int(nodes.shape[0]), seg_map)
        if _resident(t):
            return DeviceSparseTensor3(t.order, (c, nh, nw), out[:count], off[::nh].clone(), off)
        off_h = off.cpu().numpy()
        return SparseTensor3(t.order, (c, nh, nw), device.nodes_to_numpy(out, count), off_h[::nh].copy(), off_h)
    raise TypeError(f"pad_tensor does not support {type(t).__name__}")


def conv_forward_dense(t_in: DenseTensor3, filters: list[DenseTensor3], stride: int, padding: int,
                       bias: np.ndarray, workers: int = 1) -> DenseTensor3:
    """The 100%-density baseline layer (layers.py:326-342): every weight multiplied, in
    _dense_conv_kernel's order, + bias -- one bit-exact GPU launch for all filters."""
    from . import device

    geom = ConvGeometry(tuple(t_in.dims), tuple(filters[0].dims), stride, padding)
    kcrs = kernels.filters_to_device_kcrs(filters)
    b = kernels._torch().from_numpy(np.ascontiguousarray(bias, dtype=np.float32)).cuda()
    y = device.dense_conv_exact(kernels.dense_to_device(t_in), kcrs, geom.stride, geom.padding, b)
    return kernels.dense_from_device(y, _resident(t_in))
