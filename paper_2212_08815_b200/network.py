"""Network orchestration -- drop-in for the sparse-filter VGG path of sparse_infer.network.

``build_benchmark_net``, ``prepare`` and ``forward`` keep the reference's names,
signatures, validation messages and report fields (network.py:297-602).  ``prepare``
encodes every conv bank on the GPU (bit-exact SparseTensor4, as network.py:371-377)
and, for the conv3x3 -> relu [-> maxpool 2x2] stacks of ``vgg16_desk``, binds a
device-resident VGGEngine: ``forward`` then stages the whole batch (pinned H2D, GPU
layout conversion), runs one fused kernel per conv, and copies the outputs back.
Other stacks built from conv / relu / maxpool / avgpool run layer by layer through
the GPU operators in layers.py.  Batch norm, leaky ReLU, pad and the sparse-input
variant's node-format pipeline are outside the built hot path and
raise NotImplementedError.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, replace

import numpy as np

from . import layers as ly
from .sparse_core import (
    AxisOrder3,
    DenseTensor3,
    SparseTensor3,
    SparseTensor4,
    density,
)

VARIANT_SPARSE_FILTER = "sparse_filter"
VARIANT_SPARSE_INPUT = "sparse_input"
VARIANT_DENSE = "dense_baseline"
VARIANTS = (VARIANT_SPARSE_FILTER, VARIANT_SPARSE_INPUT, VARIANT_DENSE)

BENCH_KINDS = ("vgg16_desk", "yolo_desk", "vgg16_desk_noact", "yolo_desk_nobn")
_VGG16_PLAN = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
_YOLO_BLOCKS = [16, 32, 64, 128, 256]
_YOLO_HEAD = [512, 256]


@dataclass
class NetworkSpec:
    name: str
    input_dims: tuple[int, int, int]
    layers: list
    variant: str = VARIANT_DENSE

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")

    def shape_chain(self):
        dims, chain = self.input_dims, []
        for i, layer in enumerate(self.layers):
            try:
                dims = layer.out_dims(dims)
            except ValueError as e:
                raise ValueError(f"layer {i} ({layer.kind}): {e}") from None
            chain.append(dims)
        return chain

    def with_variant(self, variant: str) -> "NetworkSpec":
        return replace(self, variant=variant)


@dataclass
class ConvParams:
    filters: np.ndarray  # (K, C, H_F, W_F)
    bias: np.ndarray


@dataclass
class NetworkWeights:
    entries: list


def parameterized_layers(net: NetworkSpec):
    return [(i, l) for i, l in enumerate(net.layers) if l.kind in ("conv", "batchnorm")]


def _scaled(width: int, scale: float) -> int:
    return max(1, math.ceil(width * scale))


def build_benchmark_net(kind: str, scale: float, input_hw: int = 32, variant: str = VARIANT_DENSE) -> NetworkSpec:
    """VGG16-/YOLO-shaped stacks with scalable widths (network.py:550-602)."""
    if not 0.0 < scale <= 1.0:
        raise ValueError(f"scale must be in (0, 1], got {scale}")
    if kind not in BENCH_KINDS:
        raise ValueError(f"unknown benchmark net kind {kind!r}")
    out = []
    if kind.startswith("vgg16"):
        for item in _VGG16_PLAN:
            if item == "M":
                out.append(ly.LayerSpec(kind="maxpool", kernel=(2, 2)))
            else:
                out.append(ly.LayerSpec(kind="conv", out_channels=_scaled(item, scale), kernel=(3, 3), stride=1, padding=1))
                if kind == "vgg16_desk":
                    out.append(ly.LayerSpec(kind="relu"))
    else:
        with_bn = kind == "yolo_desk"

        def block(width):
            out.append(ly.LayerSpec(kind="conv", out_channels=_scaled(width, scale), kernel=(3, 3), stride=1, padding=1))
            if with_bn:
                out.append(ly.LayerSpec(kind="batchnorm"))
                out.append(ly.LayerSpec(kind="leaky_relu", slope=0.1))

        for width in _YOLO_BLOCKS:
            block(width)
            out.append(ly.LayerSpec(kind="maxpool", kernel=(2, 2)))
        for width in _YOLO_HEAD:
            block(width)
    net = NetworkSpec(name=kind, input_dims=(3, input_hw, input_hw), layers=out, variant=variant)
    net.shape_chain()
    return net


@dataclass
class _Step:
    layer_index: int
    kind: str
    params: object = None
    bias: np.ndarray | None = None
    stride: int = 1
    padding: int = 0
    kernel: tuple[int, int] = (0, 0)


@dataclass
class PreparedNet:
    net: NetworkSpec
    steps: list
    n_layers: int
    engine: object = None  # VGGEngine when the stack is conv3x3->relu[->maxpool2] throughout


@dataclass
class RunReport:
    variant: str
    density_setting: float
    batch: int
    workers: int
    strategy: str
    seconds: float
    layer_densities: list | None = None


@dataclass
class ForwardResult:
    outputs: list
    report: RunReport


def _vgg_plan(net: NetworkSpec):
    """The engine's plan (widths and 'M') if the stack is conv3x3/s1/p1 -> relu [-> maxpool 2x2]*."""
    layers_, plan, i = net.layers, [], 0
    c, h, w = net.input_dims
    if h != w:
        return None
    while i < len(layers_):
        l = layers_[i]
        if l.kind != "conv" or tuple(l.kernel) != (3, 3) or l.stride != 1 or l.padding != 1:
            return None
        if i + 1 >= len(layers_) or layers_[i + 1].kind != "relu":
            return None
        plan.append(l.out_channels)
        i += 2
        if i < len(layers_) and layers_[i].kind == "maxpool":
            if tuple(layers_[i].kernel) != (2, 2) or h % 2:
                return None
            plan.append("M")
            h //= 2
            i += 1
    return plan


def prepare(net: NetworkSpec, weights: NetworkWeights) -> PreparedNet:
    """Bind weights: GPU-encode every conv bank (network.py:345-407)."""
    from .sparse_core import sparsify_tensor3  # noqa: F401  (GPU encoder)

    if net.variant != VARIANT_SPARSE_FILTER:
        raise NotImplementedError(f"variant {net.variant!r} is outside the built hot path (SURVEY.md §8f-1)")
    params = dict(zip((li for li, _ in parameterized_layers(net)), weights.entries))
    steps = []
    convs = []
    for li, layer in enumerate(net.layers):
        if layer.kind == "conv":
            entry = params[li]
            if not isinstance(entry, ConvParams):
                raise ValueError(f"layer {li} expects conv parameters")
            bank = _encode_bank(np.asarray(entry.filters, np.float32))
            steps.append(_Step(li, "conv", bank, np.asarray(entry.bias, np.float32), layer.stride, layer.padding,
                               tuple(layer.kernel)))
            convs.append((np.asarray(entry.filters, np.float32), np.asarray(entry.bias, np.float32)))
        elif layer.kind in ("relu", "maxpool", "avgpool"):
            steps.append(_Step(li, layer.kind, kernel=tuple(layer.kernel)))
        else:
            raise NotImplementedError(f"layer kind {layer.kind!r} is outside the built hot path (SURVEY.md §8f)")
    engine = None
    plan = _vgg_plan(net)
    if plan is not None:
        from .engine import VGGEngine

        encoded = []
        for st in steps:
            if st.kind == "conv":
                encoded.append(st.params)
        engine = VGGEngine(None, batch=1, hw=net.input_dims[1], plan=plan, in_c=net.input_dims[0],
                           encoded=[_device_encoded(b, s.bias) for b, s in zip(encoded, [s for s in steps if s.kind == "conv"])])
    return PreparedNet(net=net, steps=steps, n_layers=len(net.layers), engine=engine)


def _encode_bank(filters: np.ndarray) -> SparseTensor4:
    """Dense (K, C, H_F, W_F) bank -> CHW SparseTensor4 via the GPU encoder."""
    import torch

    from . import device

    enc = device.encode_order(torch.from_numpy(np.ascontiguousarray(filters)).cuda(), "CHW")
    k = filters.shape[0]
    return SparseTensor4(AxisOrder3.CHW, tuple(int(v) for v in filters.shape), device.nodes_to_numpy(enc.nodes, enc.n_nodes),
                         enc.tensor_off.cpu().numpy(), enc.matrix_off.cpu().numpy().reshape(k, -1),
                         enc.seg_off.cpu().numpy().reshape(k, -1))


def _device_encoded(bank: SparseTensor4, bias: np.ndarray):
    import torch

    from . import device

    nodes = device.nodes_from_numpy(bank.nodes)
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64).ravel()).cuda()
    return (nodes, len(bank.nodes), t(bank.segment_offsets), t(bank.tensor_offsets), t(bank.matrix_offsets),
            bias, bank.count)


def prepared_from_engine(engine) -> PreparedNet:
    """Wrap an existing VGGEngine (bench.py builds it once) as a PreparedNet."""
    layers_, c = [], engine.in_c
    for item in engine.plan:
        if item == "M":
            layers_.append(ly.LayerSpec(kind="maxpool", kernel=(2, 2)))
        else:
            layers_.append(ly.LayerSpec(kind="conv", out_channels=item, kernel=(3, 3), stride=1, padding=1))
            layers_.append(ly.LayerSpec(kind="relu"))
    net = NetworkSpec("vgg16_desk", (engine.in_c, engine.hw, engine.hw), layers_, VARIANT_SPARSE_FILTER)
    return PreparedNet(net=net, steps=[], n_layers=len(layers_), engine=engine)


def _check_batch(prepared: PreparedNet, batch) -> None:
    variant = prepared.net.variant
    if not batch:
        raise ValueError("batch must be nonempty")
    for t in batch:
        if variant == VARIANT_SPARSE_INPUT:
            if not isinstance(t, SparseTensor3):
                raise ValueError(f"variant {variant} expects sparse inputs, got {type(t).__name__}")
        elif not isinstance(t, DenseTensor3):
            raise ValueError(f"variant {variant} expects dense inputs, got {type(t).__name__}")
        if tuple(t.dims) != tuple(prepared.net.input_dims):
            raise ValueError(f"input dims {t.dims} != network input {prepared.net.input_dims}")


class _Staging:
    """Pinned host buffers reused across forward calls (per batch shape)."""

    def __init__(self):
        self.key = None

    def get(self, n, in_elems, out_elems):
        import torch

        key = (n, in_elems, out_elems)
        if self.key != key:
            self.h_in = torch.empty(n * in_elems, dtype=torch.float32).pin_memory()
            self.h_out = torch.empty(n * out_elems, dtype=torch.float32).pin_memory()
            self.key = key
        return self.h_in, self.h_out


_staging = _Staging()


def _forward_engine(prepared: PreparedNet, batch) -> list:
    import torch

    from . import device

    eng = prepared.engine
    n = len(batch)
    c, h, w = prepared.net.input_dims
    oc, ohw = eng.out_c, eng.out_hw
    h_in, h_out = _staging.get(n, c * h * w, oc * ohw * ohw)
    np_in = h_in.numpy().reshape(n, -1)
    for i, t in enumerate(batch):
        np_in[i] = t.data
    d_in = h_in.to("cuda", non_blocking=True)
    x = device.whc_to_nchw(d_in, n, c, h, w)
    y = eng.forward_device(x)
    whc = device.nchw_to_whc(y.contiguous())
    h_out.copy_(whc.view(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    out = h_out.numpy().reshape(n, -1)
    return [DenseTensor3((oc, ohw, ohw), out[i].copy()) for i in range(n)]


def _run_step(step: _Step, x):
    if step.kind == "conv":
        return ly.conv_forward_strategy_II(x, step.params, step.stride, step.padding, step.bias)
    if step.kind in ("maxpool", "avgpool"):
        return ly.pool_standalone(x, step.kernel, ly.POOL_MAX if step.kind == "maxpool" else ly.POOL_AVG)
    if step.kind == "relu":
        return ly.apply_activation(x, "relu")
    raise NotImplementedError(f"step kind {step.kind!r}")


def forward(prepared: PreparedNet, batch: list, workers: int = 1,
            strategy: ly.ForwardStrategy = ly.ForwardStrategy(), record_density: bool = False,
            density_setting: float = 1.0) -> ForwardResult:
    """Run the stack over the batch and time it (network.py:478-534)."""
    _check_batch(prepared, batch)
    variant = prepared.net.variant
    strat = strategy.resolve(len(batch))
    densities = [[] for _ in range(prepared.n_layers)] if record_density else None
    t0 = time.perf_counter()
    if prepared.engine is not None and not record_density:
        outputs = _forward_engine(prepared, batch)
    else:
        if not prepared.steps:
            raise NotImplementedError("per-layer execution needs a PreparedNet from prepare()")
        outputs = []
        for t in batch:
            x = t
            for step in prepared.steps:
                x = _run_step(step, x)
                if densities is not None:
                    densities[step.layer_index].append(density(x))
            outputs.append(x)
    seconds = time.perf_counter() - t0
    layer_densities = None
    if record_density:
        layer_densities = [float(np.mean(d)) if d else float("nan") for d in densities]
    report = RunReport(variant=variant, density_setting=density_setting, batch=len(batch), workers=workers,
                       strategy=strat.name.lower() if variant == VARIANT_SPARSE_FILTER else "-",
                       seconds=seconds, layer_densities=layer_densities)
    return ForwardResult(outputs=outputs, report=report)
