"""Network orchestration -- drop-in for sparse_infer.network.

``build_benchmark_net``, ``prepare``, ``forward``, ``random_weights``,
``prune_weights`` and ``density_evolution`` keep the reference's names, signatures,
validation messages and report fields (network.py:170-643).  All three variants run
on the GPU:

* sparse_filter: ``prepare`` encodes every conv bank on the GPU (bit-exact
  SparseTensor4, network.py:371-377); for conv3x3 -> relu [-> maxpool 2x2] stacks
  (``vgg16_desk``) it binds a device-resident VGGEngine, so ``forward`` stages the
  whole batch (pinned H2D, GPU layout conversion), runs one fused kernel per conv and
  copies the outputs back;
* sparse_input: node-format activations through the sparse-input conv, node-format
  ReLU / LeakyReLU / pooling, and the conv + pool fusion rule of network.py:380-389;
* dense_baseline: the dense conv in the reference's order.
Other stacks (and density recording) run layer by layer through the GPU operators in
layers.py, exactly following the reference's step logic (network.py:410-461).
"""

from __future__ import annotations

import math
import os
import struct
import collections
import threading
import time
from dataclasses import dataclass, replace

import numpy as np

from . import layers as ly
from .sparse_core import (
    AxisOrder3,
    DenseTensor3,
    NODE_DTYPE,
    FormatError,
    SparseTensor3,
    SparseTensor4,
    dense3_from_bytes,
    dense3_to_bytes,
    density,
)

VARIANT_SPARSE_FILTER = "sparse_filter"
VARIANT_SPARSE_INPUT = "sparse_input"
VARIANT_DENSE = "dense_baseline"
VARIANTS = (VARIANT_SPARSE_FILTER, VARIANT_SPARSE_INPUT, VARIANT_DENSE)

BENCH_KINDS = ("vgg16_desk", "yolo_desk", "vgg16_desk_noact", "yolo_desk_nobn")
WEIGHT_MAGIC = b"FSNW"
WEIGHT_VERSION = 1
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
    """One runnable step; a fused conv + pool step consumes two layer indices."""

    layer_index: int
    kind: str
    params: object = None
    bias: np.ndarray | None = None
    stride: int = 1
    padding: int = 0
    kernel: tuple[int, int] = (0, 0)
    slope: float = 0.0
    fused_pool: tuple[int, int] | None = None
    fused_pool_mode: str = ly.POOL_MAX
    fused_layer_index: int = -1


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
    """Bind weights in the representation the variant needs (network.py:345-407).

    sparse_filter: GPU-encoded CHW SparseTensor4 banks; other variants: dense filter
    lists.  On sparse_input a bias-free conv directly followed by a pool whose window
    divides the conv output fuses into one step that consumes the pool layer.
    """
    params = dict(zip((li for li, _ in parameterized_layers(net)), weights.entries))
    chain = [net.input_dims] + net.shape_chain()
    steps = []
    skip = -1
    for li, layer in enumerate(net.layers):
        if li == skip:
            continue
        if layer.kind == "conv":
            entry = params[li]
            if not isinstance(entry, ConvParams):
                raise ValueError(f"layer {li} expects conv parameters")
            filters = np.asarray(entry.filters, np.float32)
            step = _Step(li, "conv", bias=np.asarray(entry.bias, np.float32), stride=layer.stride,
                         padding=layer.padding, kernel=tuple(layer.kernel))
            if net.variant == VARIANT_SPARSE_FILTER:
                step.params = _encode_bank(filters)
            else:
                step.params = [DenseTensor3.from_array(f) for f in filters]
            if net.variant == VARIANT_SPARSE_INPUT and li + 1 < len(net.layers):
                nxt = net.layers[li + 1]
                if nxt.kind in ("maxpool", "avgpool") and not np.any(step.bias != 0):
                    _, h, w = chain[li + 1]
                    h_p, w_p = nxt.kernel
                    if h % h_p == 0 and w % w_p == 0:
                        step.fused_pool = tuple(nxt.kernel)
                        step.fused_pool_mode = ly.POOL_MAX if nxt.kind == "maxpool" else ly.POOL_AVG
                        step.fused_layer_index = li + 1
                        skip = li + 1
            steps.append(step)
        elif layer.kind == "batchnorm":
            entry = params[li]
            if not isinstance(entry, ly.BatchNormParams):
                raise ValueError(f"layer {li} expects batchnorm parameters")
            entry.validate(chain[li][0])
            steps.append(_Step(li, "batchnorm", params=entry))
        else:
            steps.append(_Step(li, layer.kind, kernel=tuple(layer.kernel), padding=layer.padding,
                               slope=layer.slope))
    engine = None
    plan = _vgg_plan(net) if net.variant == VARIANT_SPARSE_FILTER else None
    if plan is not None:
        from .engine import VGGEngine

        convs = [st for st in steps if st.kind == "conv"]
        engine = VGGEngine(None, batch=1, hw=net.input_dims[1], plan=plan, in_c=net.input_dims[0],
                           encoded=[_device_encoded(st.params, st.bias) for st in convs])
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
    """Pinned host buffers reused across forward calls (per batch shape), plus a registry
    of caller-owned pinned batches (pinned_batch) that need no host-side packing."""

    def __init__(self):
        self.key = None
        # pinned_batch buffers by base address, the most recent _OWNED_MAX of them (an LRU:
        # the registry never grows without bound; an evicted batch still works, it is
        # packed into the staging buffer like any pageable batch)
        self.owned: "collections.OrderedDict[int, object]" = collections.OrderedDict()

    def get(self, n, in_elems, out_elems):
        import torch

        key = (n, in_elems, out_elems)
        if self.key != key:
            self.h_in = torch.empty(n * in_elems, dtype=torch.float32).pin_memory()
            self.h_out = torch.empty(n * out_elems, dtype=torch.float32).pin_memory()
            self.key = key
        return self.h_in, self.h_out

    def pinned_source(self, batch, elems):
        """The pinned tensor holding the batch back to back (zero-copy H2D), or None."""
        addr = [t.data.__array_interface__["data"][0] for t in batch]
        nbytes = elems * 4
        tensor = self.owned.get(addr[0])
        if tensor is not None and len(batch) * nbytes <= tensor.numel() * 4 and all(
                a == addr[0] + i * nbytes for i, a in enumerate(addr)):
            self.owned.move_to_end(addr[0])
            return tensor[: len(batch) * elems]
        return None

    def register(self, buf) -> None:
        self.owned[buf.data_ptr()] = buf
        while len(self.owned) > _OWNED_MAX:
            self.owned.popitem(last=False)


_OWNED_MAX = 16
_staging = _Staging()
# forward() may be called from several host threads (the reference's kernels are nogil
# and its API thread-safe); the engine's device buffers and the pinned staging above are
# shared per process, so engine forwards are serialised.
_engine_lock = threading.Lock()


def pinned_batch(n: int, dims) -> list:
    """n zeroed DenseTensor3 of ``dims`` whose payloads live back to back in one pinned
    host buffer: filling these and passing the list to ``forward`` lets the input go to
    the GPU with one DMA and no host-side packing (the usual pinned-staging practice;
    any other list of DenseTensor3 works too, it is packed into pinned memory first)."""
    import torch

    c, h, w = dims
    elems = c * h * w
    buf = torch.zeros(n * elems, dtype=torch.float32).pin_memory()
    _staging.register(buf)
    arr = buf.numpy().reshape(n, elems)
    return [DenseTensor3((c, h, w), arr[i]) for i in range(n)]


def _engine_device_forward(prepared: PreparedNet, batch):
    """Host DenseTensor3 batch -> the engine's device (W,H,C) output [n, W', H', C']
    (pinned H2D in parts overlapped with the first conv; the caller holds _engine_lock)."""
    eng = prepared.engine
    n = len(batch)
    c, h, w = prepared.net.input_dims
    elems = c * h * w
    h_in, _ = _staging.get(n, elems, eng.out_c * eng.out_hw * eng.out_hw)
    src = _staging.pinned_source(batch, elems)
    fill = None
    if src is None:  # pageable inputs: pack each half into pinned staging just before its copy
        np_in = h_in.numpy().reshape(n, elems)

        def fill(lo, hi):
            # on host threads (numpy copies release the GIL)
            def pack(i):
                np_in[i] = batch[i].data

            if hi - lo > 1:
                list(_pack_pool().map(pack, range(lo, hi)))
            else:
                for i in range(lo, hi):
                    pack(i)

        src = h_in
    if ly._EXACT:  # set_exact(True): the reference-order kernels, bit-exact
        return eng.forward_from_host_exact(src, n, fill)
    return eng.forward_from_host(src, n, fill)


def _whc_to_host(whc, n: int, oc: int, ohw: int) -> list:
    """Device (W,H,C) outputs -> host DenseTensor3 list (one D2H into fresh pinned memory;
    torch's caching host allocator recycles it once the returned arrays are gone)."""
    import torch

    res = torch.empty(n * oc * ohw * ohw, dtype=torch.float32, pin_memory=True)
    res.copy_(whc.reshape(-1), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    out = res.numpy().reshape(n, -1)
    return [DenseTensor3((oc, ohw, ohw), out[i]) for i in range(n)]


def _forward_engine(prepared: PreparedNet, batch) -> list:
    eng = prepared.engine
    whc = _engine_device_forward(prepared, batch)
    return _whc_to_host(whc, len(batch), eng.out_c, eng.out_hw)


_BATCHED = True  # tests switch it off to compare against the per-image layer path


def _batched_inputs_ok(prepared: PreparedNet, batch) -> bool:
    """The batched device path covers all three variants for inputs the per-image path
    would accept unchanged (sparse_input: CHW node tensors without explicit zero-valued
    nodes -- the batch travels as dense device planes, where a stored zero and an absent
    node coincide); anything else takes the per-image path and its validation.
    (The zero-valued-node test runs on the device inside _forward_batched, which then
    declines the batch.)"""
    variant = prepared.net.variant
    if not prepared.steps:
        return False
    if variant == VARIANT_SPARSE_INPUT:
        return all(t.order is AxisOrder3.CHW for t in batch)
    return True


_pinned_in: dict = {}  # grow-only pinned staging for the sparse-input batch upload
_pinned_lock = threading.Lock()  # forward() may run on several host threads


def _pinned(key: str, nbytes: int):
    import torch

    buf = _pinned_in.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1), dtype=torch.uint8, pin_memory=True)
        _pinned_in[key] = buf
    return buf


def _upload_sparse_batch(batch, c: int, h: int, w: int, dev):
    """The batch's CHW node tensors as one device node buffer + global segment offsets
    (packed into pinned staging on host threads, one H2D each), or None -- the caller
    then takes the per-image path -- when a stored node has value +-0.0 (the dense
    batched path cannot represent it) or the structure is not the reference format's
    (both checked on the device)."""
    with _pinned_lock:  # the staging is reused: held until the copies have completed
        return _upload_sparse_batch_locked(batch, c, h, w, dev)


_pack_pool_obj = None


def _pack_pool():
    global _pack_pool_obj
    if _pack_pool_obj is None:
        import concurrent.futures

        _pack_pool_obj = concurrent.futures.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4))
    return _pack_pool_obj


def _upload_sparse_batch_locked(batch, c: int, h: int, w: int, dev):
    import torch

    # shapes the dense batched path cannot take (the per-image path validates and reports)
    if any(np.asarray(t.nodes).dtype != NODE_DTYPE or len(t.segment_offsets) != h * w for t in batch):
        return None
    arrs = [np.asarray(t.nodes).view(np.int32).reshape(-1, 2) for t in batch]
    counts = np.array([a.shape[0] for a in arrs], np.int64)
    total = int(counts.sum())
    hn = _pinned("nodes", total * 8)[: total * 8].view(torch.int32).view(-1, 2)
    hs = _pinned("seg", len(batch) * h * w * 8)[: len(batch) * h * w * 8].view(torch.int64).view(len(batch), h * w)
    # pack on host threads (numpy copies release the GIL): ~9 ms -> ~2 ms at batch 32
    starts = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    hn_np, hs_np = hn.numpy(), hs.numpy()

    def pack(i):
        hn_np[starts[i]:starts[i + 1]] = arrs[i]
        hs_np[i] = batch[i].segment_offsets

    list(_pack_pool().map(pack, range(len(batch))))
    nodes = torch.empty((max(total, 1), 2), dtype=torch.int32, device=dev)
    if total:
        nodes[:total].copy_(hn, non_blocking=True)
    seg = hs.to(dev, non_blocking=True)
    base = torch.from_numpy(np.concatenate([[0], np.cumsum(counts)[:-1]]).astype(np.int64)).to(dev)
    seg += base.view(-1, 1)
    # one device check, one sync: a stored zero (index >= 0, value bits +-0.0) cannot
    # travel as a dense plane, and the structure must be what the decoder walks (each
    # segment's channels ascending in [0, c), its sentinel right before the next
    # segment's offset); otherwise the per-image path runs and its validate() reports
    seg = seg.view(-1)
    if not total:
        torch.cuda.current_stream().synchronize()  # the pinned staging is free again
        return None
    idx = nodes[:total, 0]
    bad = ((idx >= 0) & ((nodes[:total, 1] & 0x7FFFFFFF) == 0)).any()
    bad |= (idx >= c).any() | (idx < -1).any() | (idx[total - 1] != -1)
    bad |= ((idx[1:] <= idx[:-1]) & (idx[1:] >= 0) & (idx[:-1] >= 0)).any()
    bad |= (seg[0] != 0) | (seg[1:] <= seg[:-1]).any() | (seg[-1] >= total)
    bad |= (idx[(seg[1:] - 1).clamp(0, total - 1)] != -1).any()
    bad |= (idx == -1).sum() != seg.numel()
    if bool(bad):
        return None
    return nodes[:total], seg


def _step_bias(step: _Step, dev):
    """The step's bias on the device (cached on the step)."""
    import torch

    b = getattr(step, "_dev_bias", None)
    if b is None:
        b = step._dev_bias = torch.from_numpy(np.ascontiguousarray(step.bias, np.float32)).to(dev)
    return b


def _step_bank(step: _Step, kind: str):
    """A device re-layout of the step's filters for one sparse-input kernel ('fast',
    'strip' or 'gather'), packed once and cached on the step."""
    from . import device

    banks = getattr(step, "_dev_banks", None)
    if banks is None:
        banks = step._dev_banks = {}
    if kind not in banks:
        pack = {"fast": device.si_pack_fast, "strip": device.si_pack3x3, "gather": device.kcrs_to_crsk}[kind]
        banks[kind] = pack(_step_filters(step))
    return banks[kind]


def _step_filters(step: _Step):
    """Device copies of a conv step's filters (cached on the step): [K, C, R, S]."""
    cache = getattr(step, "_dev_filters", None)
    if cache is None:
        from . import kernels

        cache = kernels.filters_to_device_kcrs(step.params)
        step._dev_filters = cache
    return cache


def _forward_batched(prepared: PreparedNet, batch, densities=None) -> list:
    """All images of the batch through the layer stack at once, activations resident in
    HBM between steps (dense [N, C, H, W] planes; node-format steps are the same
    decode -> op -> re-encode the per-image operators do, so each image's result is the
    per-image result, bit for bit: every kernel is batch-position invariant and the
    sparse-input kernel is chosen by the per-image rule).  With ``densities`` (one list
    per layer) each step's per-image density is appended, as density() of the per-image
    output would give it (stored nodes = nonzeros of the plane)."""
    import torch

    from . import device
    from .kernels import ConvGeometry

    variant = prepared.net.variant
    n = len(batch)
    c, h, w = prepared.net.input_dims
    dev = torch.device("cuda", torch.cuda.current_device())
    if variant == VARIANT_SPARSE_INPUT:
        up = _upload_sparse_batch(batch, c, h, w, dev)
        if up is None:
            return None
        x = device.decode_order(up[0], up[1], (n, c, h, w), "CHW")
        sparse = True
    else:
        whc = torch.from_numpy(np.stack([np.asarray(t.data, np.float32) for t in batch])).to(dev)
        x = device.whc_to_nchw(whc.view(-1), n, c, h, w)
        sparse = False
    counts = []  # (step, per-image nonzero counts on the device)
    for step in prepared.steps:
        dims = tuple(int(v) for v in x.shape[1:])
        if step.kind == "conv":
            if variant == VARIANT_SPARSE_FILTER:
                kcrs = None
                k, c_f, h_f, w_f = (int(v) for v in step.params.dims)
            else:
                kcrs = _step_filters(step)
                k, c_f, h_f, w_f = (int(v) for v in kcrs.shape)
            geom = ConvGeometry(dims, (c_f, h_f, w_f), step.stride, step.padding)
            bias = _step_bias(step, dev)
            if sparse:
                _, ci, hi, wi = (int(v) for v in x.shape)
                fused = False
                if (h_f, w_f, step.stride, step.padding) == (3, 3, 1, 1) and not ly._EXACT and \
                        device.si_use_fast(hi, wi, k):
                    # Alg. 7 in the kernel's epilogue when the fused pool is 2x2 (VGG16's)
                    fp = None
                    if step.fused_pool is not None and tuple(step.fused_pool) == (2, 2) and hi % 2 == 0 \
                            and wi % 2 == 0:
                        fp = "max" if step.fused_pool_mode == ly.POOL_MAX else "avg"
                    # straight from the dense activation: the same tile streams as encoding it
                    # (bit-identical), without the encode and its host sync
                    y = device.si_conv3x3_fast_dense(x, _step_bank(step, "fast"), k, pool=fp)
                    fused = fp is not None
                else:
                    enc = device.encode_order(x, "CHW")
                    if (h_f, w_f, step.stride, step.padding) == (3, 3, 1, 1):
                        y = device.si_conv3x3(enc.nodes, enc.seg_off, n, ci, hi, wi, _step_bank(step, "strip"), k)
                    else:
                        y = device.si_conv(enc.nodes, enc.seg_off, n, ci, hi, wi, _step_bank(step, "gather"), k,
                                           h_f, w_f, step.stride, step.padding)
                if step.fused_pool is not None and not fused:
                    h_p, w_p = ly._pool_args(step.fused_pool, step.fused_pool_mode, geom.n_h, geom.n_w)
                    y = device.pool2d(y, h_p, w_p, step.fused_pool_mode == ly.POOL_MAX)
                if np.any(step.bias != 0):
                    y = y + bias.view(1, -1, 1, 1)
                    sparse = False
            elif variant == VARIANT_SPARSE_FILTER:
                # the strategy I / II layer (layers._sf_layer), all images in one launch
                nodes, seg, packed = ly._device_bank(step.params)
                if packed is not None and (step.stride, step.padding) == (1, 1) and not ly._EXACT:
                    y = device.sf_conv3x3(device.to_halo(x), packed, bias, relu=False, pool=False, w=dims[2])
                    y = device.from_halo(y, dims[2]).contiguous()
                else:
                    y = device.sf_conv_exact(x, nodes, seg, k, h_f, w_f, step.stride, step.padding, bias)
            else:
                y = device.dense_conv_exact(x, kcrs, step.stride, step.padding, bias)
                if step.fused_pool is not None:
                    h_p, w_p = ly._pool_args(step.fused_pool, step.fused_pool_mode, geom.n_h, geom.n_w)
                    y = device.pool2d(y, h_p, w_p, step.fused_pool_mode == ly.POOL_MAX)
            x = y
        elif step.kind in ("maxpool", "avgpool"):
            h_p, w_p = step.kernel
            if h_p <= 0 or w_p <= 0:
                raise ValueError(f"pool window must be positive, got {step.kernel}")
            if dims[1] % h_p or dims[2] % w_p:
                raise ValueError(f"input {dims[1]}x{dims[2]} not divisible by pool window {h_p}x{w_p}")
            x = device.pool2d(x, h_p, w_p, step.kind == "maxpool")
        elif step.kind in ("relu", "leaky_relu"):
            if step.slope < 0:
                raise ValueError("leaky slope must be non-negative")
            if step.kind == "relu":
                kind = device.ACT_RELU_NODES if sparse else device.ACT_RELU
            else:
                kind = device.ACT_LEAKY
            x = device.activation(x, kind, step.slope)
        elif step.kind == "batchnorm":
            prm = step.params
            prm.validate(dims[0])
            x = device.batchnorm(x, prm.scale, prm.shift, prm.mean, prm.var, prm.epsilon)
        elif step.kind == "pad":
            if step.padding < 0:
                raise ValueError("pad width must be non-negative")
            if step.padding:
                x = device.pad2d(x, step.padding)
        else:
            raise ValueError(f"unknown step kind {step.kind!r}")
        if densities is not None:
            counts.append((step, torch.count_nonzero(x.reshape(n, -1), dim=1), x[0].numel()))
    for step, cnt, size in counts:
        for v in cnt.cpu().tolist():
            d = float(v) / float(size)
            densities[step.layer_index].append(d)
            if step.fused_layer_index >= 0:
                densities[step.fused_layer_index].append(d)
    oc, oh, ow = (int(v) for v in x.shape[1:])
    if sparse:
        enc = device.encode_order(x, "CHW")
        nodes_h = device.nodes_to_numpy(enc.nodes, enc.n_nodes)
        seg_h = enc.seg_off.cpu().numpy().reshape(n, ow * oh)
        ten_h = np.append(enc.tensor_off.cpu().numpy(), enc.n_nodes)
        outs = []
        for i in range(n):
            lo, hi_ = int(ten_h[i]), int(ten_h[i + 1])
            so = seg_h[i] - lo
            outs.append(SparseTensor3(AxisOrder3.CHW, (oc, oh, ow), nodes_h[lo:hi_].copy(), so[::oh].copy(), so))
        return outs
    whc = device.nchw_to_whc(x).cpu().numpy().reshape(n, -1)
    return [DenseTensor3((oc, oh, ow), whc[i].copy()) for i in range(n)]


def _run_step(step: _Step, x, variant: str, strat):
    """One step (network.py:410-448), every branch a GPU operator."""
    if step.kind == "conv":
        if isinstance(x, SparseTensor3):
            return ly.conv_forward_sparse_input(x, step.params, step.stride, step.padding, step.bias,
                                                fused_pool=step.fused_pool, pool_mode=step.fused_pool_mode)
        if variant == VARIANT_SPARSE_FILTER:
            if strat is ly.StrategyKind.STRATEGY_I:
                return ly.conv_forward_strategy_I(x, step.params, step.stride, step.padding, step.bias)
            return ly.conv_forward_strategy_II(x, step.params, step.stride, step.padding, step.bias)
        out = ly.conv_forward_dense(x, step.params, step.stride, step.padding, step.bias)
        if step.fused_pool is not None:
            # an upstream biased conv turned the pipeline dense; the consumed pool still runs
            out = ly.pool_standalone(out, step.fused_pool, step.fused_pool_mode)
        return out
    if step.kind in ("maxpool", "avgpool"):
        mode = ly.POOL_MAX if step.kind == "maxpool" else ly.POOL_AVG
        if isinstance(x, SparseTensor3):
            return ly.pool_sparse(x, step.kernel, mode)
        return ly.pool_standalone(x, step.kernel, mode)
    if step.kind in ("relu", "leaky_relu"):
        return ly.apply_activation(x, step.kind, step.slope)
    if step.kind == "batchnorm":
        return ly.apply_batchnorm(x, step.params)
    if step.kind == "pad":
        return ly.pad_tensor(x, step.padding)
    raise ValueError(f"unknown step kind {step.kind!r}")


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
        with _engine_lock:
            outputs = _forward_engine(prepared, batch)
    else:
        outputs = _forward_batched(prepared, batch, densities) \
            if _BATCHED and _batched_inputs_ok(prepared, batch) else None
    if outputs is None:
        if not prepared.steps:
            raise NotImplementedError("per-layer execution needs a PreparedNet from prepare()")
        outputs = []
        for t in batch:
            x = t
            for step in prepared.steps:
                x = _run_step(step, x, variant, strat)
                if densities is not None:
                    densities[step.layer_index].append(density(x))
                    if step.fused_layer_index >= 0:
                        # the conv intermediate never materialises: both layers see the pool
                        densities[step.fused_layer_index].append(density(x))
            outputs.append(x)
    seconds = time.perf_counter() - t0
    layer_densities = None
    if record_density:
        layer_densities = [float(np.mean(d)) if d else float("nan") for d in densities]
    report = RunReport(variant=variant, density_setting=density_setting, batch=len(batch), workers=workers,
                       strategy=strat.name.lower() if variant == VARIANT_SPARSE_FILTER else "-",
                       seconds=seconds, layer_densities=layer_densities)
    return ForwardResult(outputs=outputs, report=report)


# -- weights and the density-evolution study (network.py:170-207, :605-643) ----------


def random_weights(net: NetworkSpec, seed: int) -> NetworkWeights:
    """Filters uniform on [-0.5, 0.5], zero biases, batch-norm statistics uniform with
    var in [0.5, 1.5]; one numpy generator per layer seeded [seed, layer] (host-side
    workload generation, draw order as network.py:173-195)."""
    chain = [net.input_dims] + net.shape_chain()
    entries = []
    for li, layer in parameterized_layers(net):
        rng = np.random.default_rng([seed, li])
        c_in = chain[li][0]
        if layer.kind == "conv":
            shape = (layer.out_channels, c_in) + tuple(layer.kernel)
            entries.append(ConvParams(filters=rng.uniform(-0.5, 0.5, shape).astype(np.float32),
                                      bias=np.zeros(layer.out_channels, np.float32)))
        else:
            draws = [rng.uniform(lo, hi, c_in).astype(np.float32)
                     for lo, hi in ((0.5, 1.5), (-0.5, 0.5), (-0.5, 0.5), (0.5, 1.5))]
            entries.append(ly.BatchNormParams(scale=draws[0], shift=draws[1], mean=draws[2], var=draws[3],
                                              epsilon=1e-5))
    return NetworkWeights(entries=entries)


def prune_weights(weights: NetworkWeights, target_density: float, seed: int) -> NetworkWeights:
    """Prune every conv bank jointly to the target density, generator [seed, entry]."""
    from .sparse_core import prune_array

    out = []
    for i, entry in enumerate(weights.entries):
        if isinstance(entry, ConvParams):
            out.append(ConvParams(filters=prune_array(entry.filters, target_density, [seed, i]), bias=entry.bias))
        else:
            out.append(entry)
    return NetworkWeights(entries=out)


@dataclass
class DensityRecord:
    input_density: float
    layer_index: int
    layer_kind: str
    output_density: float


def random_input(dims, seed: int) -> DenseTensor3:
    rng = np.random.default_rng([seed, 0xBA7C4])
    return DenseTensor3.from_array(rng.uniform(-0.5, 0.5, dims).astype(np.float32))


def density_evolution(net: NetworkSpec, input_density_sweep: list, seed: int) -> list:
    """Per-layer output densities for each input density (network.py:621-643): record 0
    is the pruned input, record i+1 the output of layer i -- every layer on the GPU."""
    from .sparse_core import prune_random, sparsify_tensor3

    if net.variant != VARIANT_SPARSE_INPUT:
        raise ValueError("density evolution requires the sparse_input variant")
    prepared = prepare(net, random_weights(net, seed))
    base = random_input(net.input_dims, seed)
    records = []
    for d in input_density_sweep:
        sp = sparsify_tensor3(prune_random(base, d, seed), AxisOrder3.CHW)
        records.append(DensityRecord(d, 0, "input", density(sp)))
        result = forward(prepared, [sp], record_density=True)
        for li, layer in enumerate(net.layers):
            records.append(DensityRecord(d, li + 1, layer.kind, result.report.layer_densities[li]))
    return records


# -- model text and FSNW weight files (network.py:99-167, :210-294): host-side I/O -------


def parse_model_text(text: str, name: str = "model") -> NetworkSpec:
    """Line-oriented model format: ``input c= h= w=`` then one layer per line
    (conv out= k= [s=] [p=], maxpool/avgpool k=, relu, leaky_relu slope=, batchnorm,
    pad p=); '#' starts a comment."""
    dims, stack = None, []
    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        kind, *fields = line.split()
        args = {}
        for f in fields:
            key, sep, val = f.partition("=")
            if not sep:
                raise FormatError(f"line {lineno}: malformed key=value field")
            args[key] = val
        try:
            if kind == "input":
                dims = (int(args["c"]), int(args["h"]), int(args["w"]))
            elif kind == "conv":
                k = int(args["k"])
                stack.append(ly.LayerSpec(kind="conv", out_channels=int(args["out"]), kernel=(k, k),
                                          stride=int(args.get("s", 1)), padding=int(args.get("p", 0))))
            elif kind in ("maxpool", "avgpool"):
                k = int(args["k"])
                stack.append(ly.LayerSpec(kind=kind, kernel=(k, k)))
            elif kind in ("relu", "batchnorm"):
                stack.append(ly.LayerSpec(kind=kind))
            elif kind == "leaky_relu":
                stack.append(ly.LayerSpec(kind="leaky_relu", slope=float(args["slope"])))
            elif kind == "pad":
                stack.append(ly.LayerSpec(kind="pad", padding=int(args["p"])))
            else:
                raise FormatError(f"line {lineno}: unknown layer kind {kind!r}")
        except (KeyError, ValueError) as e:
            raise FormatError(f"line {lineno}: {e}") from None
    if dims is None:
        raise FormatError("model text is missing an 'input c= h= w=' line")
    net = NetworkSpec(name=name, input_dims=dims, layers=stack)
    net.shape_chain()
    return net


def format_model_text(net: NetworkSpec) -> str:
    c, h, w = net.input_dims
    out = [f"input c={c} h={h} w={w}"]
    for l in net.layers:
        if l.kind == "conv":
            out.append(f"conv out={l.out_channels} k={l.kernel[0]} s={l.stride} p={l.padding}")
        elif l.kind in ("maxpool", "avgpool"):
            out.append(f"{l.kind} k={l.kernel[0]}")
        elif l.kind == "leaky_relu":
            out.append(f"leaky_relu slope={l.slope:g}")
        elif l.kind == "pad":
            out.append(f"pad p={l.padding}")
        else:
            out.append(l.kind)
    return "\n".join(out) + "\n"


def save_weights(path, net: NetworkSpec, weights: NetworkWeights) -> None:
    """FSNW file: magic, u32 version, u32 entry count, then per parameterized layer --
    conv: u32 K, C, H_F, W_F, K FDT3 filter blobs, K f32 biases; batchnorm: C f32 each of
    scale, shift, mean, var, then f32 epsilon (little endian)."""
    params = parameterized_layers(net)
    if len(params) != len(weights.entries):
        raise ValueError(f"{len(weights.entries)} entries for {len(params)} parameterized layers")
    blob = bytearray(WEIGHT_MAGIC + struct.pack("<II", WEIGHT_VERSION, len(params)))
    for (_, layer), entry in zip(params, weights.entries):
        if layer.kind == "conv":
            filters = np.asarray(entry.filters, np.float32)
            blob += struct.pack("<IIII", *filters.shape)
            for f in filters:
                blob += dense3_to_bytes(DenseTensor3.from_array(f))
            blob += np.asarray(entry.bias, dtype="<f4").tobytes()
        else:
            for arr in (entry.scale, entry.shift, entry.mean, entry.var):
                blob += np.asarray(arr, dtype="<f4").tobytes()
            blob += struct.pack("<f", entry.epsilon)
    with open(path, "wb") as fh:
        fh.write(bytes(blob))


def load_weights(path, net: NetworkSpec) -> NetworkWeights:
    """Read an FSNW file and validate it against the layer stack (same messages as the
    reference: magic, version, entry count, dims, truncation, trailing bytes)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw[:4] != WEIGHT_MAGIC:
        raise FormatError(f"bad magic {raw[:4]!r}, expected {WEIGHT_MAGIC!r}")
    if len(raw) < 12:
        raise FormatError("truncated weight file header")
    version, count = struct.unpack_from("<II", raw, 4)
    if version != WEIGHT_VERSION:
        raise FormatError(f"unsupported weight file version {version}")
    params = parameterized_layers(net)
    if count != len(params):
        raise FormatError(f"weight file has {count} parameterized layers, network expects {len(params)}")
    chain = [net.input_dims] + net.shape_chain()
    at = 12
    entries = []

    def need(n, where):
        if at + n > len(raw):
            raise FormatError(f"truncated weight file in {where}")

    for li, layer in params:
        where = f"layer {li} ({layer.kind})"
        if layer.kind == "conv":
            need(16, where)
            dims = struct.unpack_from("<IIII", raw, at)
            at += 16
            expect = (layer.out_channels, chain[li][0]) + tuple(layer.kernel)
            if tuple(dims) != expect:
                raise FormatError(f"filter dims {tuple(dims)} != {expect} in {where}")
            k, c, h, w = dims
            per = 16 + 4 * c * h * w
            filters = np.empty(dims, np.float32)
            for f in range(k):
                need(per, where)
                t = dense3_from_bytes(raw[at:at + per])
                if tuple(t.dims) != (c, h, w):
                    raise FormatError(f"filter {f} dims {t.dims} != {(c, h, w)} in {where}")
                filters[f] = t.to_array()
                at += per
            need(4 * k, where)
            bias = np.frombuffer(raw, dtype="<f4", count=k, offset=at).astype(np.float32)
            at += 4 * k
            entries.append(ConvParams(filters=filters, bias=bias))
        else:
            c_in = chain[li][0]
            need(16 * c_in + 4, where)
            stats = []
            for _ in range(4):
                stats.append(np.frombuffer(raw, dtype="<f4", count=c_in, offset=at).astype(np.float32))
                at += 4 * c_in
            (eps,) = struct.unpack_from("<f", raw, at)
            at += 4
            entries.append(ly.BatchNormParams(scale=stats[0], shift=stats[1], mean=stats[2], var=stats[3],
                                              epsilon=float(eps)))
    if at != len(raw):
        raise FormatError(f"{len(raw) - at} trailing bytes after last layer")
    return NetworkWeights(entries=entries)
