"""Device-resident VGG16-shaped sparse-filter conv stack (the BASELINE config 3/5 path).

Mirrors network.prepare + network.forward for the ``vgg16_desk`` stack in the
``sparse_filter`` variant (network.py:345-407, :410-534, plan :541): 13 3x3/s1/p1
convs, ReLU after each, 2x2 max-pool after each block.  On the device every
conv -> ReLU [-> max-pool] group is ONE launch of the fast sparse-filter kernel
(ReLU and pool fused into its epilogue, in the reference's relu -> pool order), and
activations stay in HBM between layers in NCHW "halo-column" buffers (logical column j
at memory column j+1, zero columns around it, 16-byte row pitch) so every TMA box the
kernel loads starts 16-byte aligned.

Preparation encodes each dense filter bank on the GPU into the reference's CHW
SparseTensor4 node format (kept, bit-exact with sparsify_tensor3 + stack) and packs
it into the kernel's channel-major stream.  Multi-GPU runs replicate the encoded
banks (see distributed.py) and shard the batch.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import device
from .workloads import VGG16_PLAN


@dataclass
class ConvStep:
    k: int
    c: int
    h: int
    w: int
    pool: bool
    bank: device.PackedBank
    bias: torch.Tensor
    nodes: torch.Tensor      # reference CHW node buffer (SparseTensor4.nodes)
    seg_off: torch.Tensor    # SparseTensor4.segment_offsets, [K*9]
    tensor_off: torch.Tensor
    matrix_off: torch.Tensor
    n_nodes: int
    ly: int = 0
    small: dict | None = None  # kt -> packed stream with 1 / 2 filters per warp (small grids)
    jit: device.SfJit | None = None  # the bank compiled into per-group kernels (sfjit.cu)

    def conv(self, x: torch.Tensor, out: torch.Tensor, w: int, n_plan: int) -> torch.Tensor:
        """conv3x3 + bias + ReLU [+ 2x2 max-pool] of a halo-column batch into ``out``:
        the specialised kernels when compiled, else the jump-table kernel (identical bits)."""
        if self.jit is not None and n_plan >= SFJIT_MIN_BATCH:
            return self.jit(x, out=out)
        bank, warps = self.plan_for(n_plan)
        return device.sf_conv3x3(x, bank, self.bias, relu=True, pool=self.pool, out=out, w=w, ly=self.ly,
                                 cta_warps=warps)

    def plan_for(self, n: int) -> tuple[device.PackedBank, int]:
        """(packed stream, warps per CTA) for a launch over n images: fewer filters per
        warp when the 4-filter grid leaves SMs idle (bit-identical results either way)."""
        if self.small:
            kt, warps = device.sf_grid_plan(n, self.h, self.w, self.k, self.ly)
            if kt in self.small:
                return self.small[kt], warps
        return self.bank, 0


# Below this batch the jump-table kernel's small-grid plans win (a specialised kernel
# CTA walks its group's whole code once however few tiles it has: VGG16 batch 1
# 0.91 vs 1.46 ms, batch 8 2.30 vs 2.58; batch 16: 4.03 vs 3.10); the compiled code
# does not depend on the batch, so both stay ready.
SFJIT_MIN_BATCH = int(os.environ.get("FSCNN_SFJIT_MIN_BATCH", "12"))


def _align4(v: int) -> int:
    return (v + 3) // 4 * 4


class VGGEngine:
    """Prepared VGG16 conv stack on one GPU.

    layers: list of (filters (K, C, 3, 3) float32, bias (K,)) in plan order -- numpy
    arrays (uploaded here) or CUDA tensors; or pre-encoded banks via ``from_encoded``.
    """

    def __init__(self, layers, batch: int, hw: int = 224, plan=VGG16_PLAN, in_c: int = 3,
                 encoded=None, jit: bool | None = None):
        self.batch, self.hw, self.plan = batch, hw, list(plan)
        self.in_c = in_c
        if jit is None:
            jit = device.sfjit_enabled()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.steps: list[ConvStep] = []
        c, h = in_c, hw
        li = 0
        conv_idx = [i for i, it in enumerate(self.plan) if it != "M"]
        for pos in conv_idx:
            pool = pos + 1 < len(self.plan) and self.plan[pos + 1] == "M"
            if encoded is not None:
                nodes, n_nodes, seg, ten, mat, bias_np, k = encoded[li]
                dense = torch.empty((k, c, 3, 3), dtype=torch.float32, device=dev)
                device.decode(nodes, seg, k, 3, 3, c, dense, (c * 9, 1, 3, 9))
                bias_t = torch.as_tensor(np.asarray(bias_np, np.float32)).to(dev)
            else:
                filt, bias_np = layers[li]
                dense = torch.as_tensor(np.asarray(filt, np.float32) if not torch.is_tensor(filt) else filt)
                dense = dense.to(dev, torch.float32).contiguous()
                k = int(dense.shape[0])
                assert tuple(dense.shape[1:]) == (c, 3, 3), (dense.shape, c)
                enc = device.encode_order(dense, "CHW")
                nodes, n_nodes, seg, ten, mat = enc.nodes, enc.n_nodes, enc.seg_off, enc.tensor_off, enc.matrix_off
                bias_t = torch.as_tensor(np.asarray(bias_np, np.float32) if not torch.is_tensor(bias_np) else bias_np)
                bias_t = bias_t.to(dev, torch.float32).contiguous()
            bank = device.sf_pack(dense)
            small = {kt: device.sf_pack(dense, kt) for kt in (1, 2)} if bank.kt == 4 else None
            step = ConvStep(k, c, h, h, pool, bank, bias_t, nodes, seg, ten, mat, n_nodes, device.pick_ly(c, h), small)
            if jit and h % 2 == 0:
                # compile jobs are submitted here and run on host threads while the next
                # banks are encoded; the first forward joins them
                # 48 filters per group: the whole stack's best with its batch parts running
                # concurrently (the layer-alone density rule of sfjit.cu's pick_flags, 64 at
                # <= 7 % density, measured 10 % slower per C5 step although each layer alone
                # runs faster)
                # ... except the shallow layers (C <= 64), run outside the batch parts (or per
                # H2D part): 64-filter groups there (alone L1 -14 %, L2 -10 %;
                # profiles/r02_sfjit_kt90.txt)
                kt = 0 if os.environ.get("FSCNN_SFJIT_KT") else \
                    (int(os.environ.get("FSCNN_SFJIT_SHALLOW_KT", "64")) if c <= 64 else 48)
                step.jit = device.SfJit(dense, bias_t, h, h, relu=True, pool=pool, flags=kt)
            self.steps.append(step)
            c = k
            if pool:
                h //= 2
            li += 1
        self.out_c, self.out_hw = c, h
        # batch split over streams: helps the jump-table kernel's partial last waves; the
        # specialised kernels already spread each layer over concurrent per-group launches
        # batch split over concurrent streams: with the specialised kernels a layer's code
        # is fetched from HBM by the first part and found in L2 by the others, and one
        # part's partial last wave overlaps another's next layer (VGG16 @224, batch 32,
        # replayed as a graph: 1 part 4.79 ms, 2: 4.08, 4: 3.74, 8: 3.70;
        # tools/stack_probe.py)
        self._jit_all = all(st.jit is not None for st in self.steps)
        self.use_graphs = os.environ.get("FSCNN_GRAPHS", "1") != "0"
        self._graphs = {}
        self._bufs = None
        self._bufs_batch = None

    # -- buffers ------------------------------------------------------------------------
    def _buffers(self, n: int):
        if self._bufs is None or self._bufs_batch != n:
            dev = torch.device("cuda", torch.cuda.current_device())
            self._in = device.halo_empty(n, self.in_c, self.hw, self.hw, dev)
            bufs = []
            for st in self.steps:
                ho = st.h // 2 if st.pool else st.h
                bufs.append(device.halo_empty(n, st.k, ho, ho, dev))
            self._bufs, self._bufs_batch = bufs, n
            self._graphs.clear()  # captured graphs point at the old buffers
        return self._bufs

    @property
    def launches_per_forward(self) -> int:
        return len(self.steps)

    def stage_input(self, x: torch.Tensor) -> torch.Tensor:
        """Copy a dense [N, C, H, W] CUDA batch into the engine's halo input buffer."""
        self._buffers(int(x.shape[0]))
        return device.nchw_into_halo(x, self._in)

    def run(self, xh: torch.Tensor, parts: int | None = None) -> torch.Tensor:
        """Run the stack on a halo-layout input; returns the halo output buffer.

        The batch is split over ``parts`` streams, each walking all layers on its slice:
        one slice's last (partial) wave of a layer overlaps the other slice's next layer,
        instead of leaving SMs idle at every layer boundary (measured -5 % on the VGG16
        stack at batch 32).  Results are identical (the kernels are batch-position
        invariant).
        """
        return self._run(0, xh, self.parts_for(int(xh.shape[0])) if parts is None else parts)

    def parts_for(self, n: int) -> int:
        if os.environ.get("FSCNN_PARTS"):
            return int(os.environ["FSCNN_PARTS"])
        if not (self._jit_all and n >= SFJIT_MIN_BATCH):
            return 2
        # more parts = later parts find the code earlier ones fetched (C3 @ 32: 4 -> 8
        # parts 8.73k -> 8.82k img/s; C5 @ 256: 8 -> 16 parts 12.4k -> 14.2k img/s)
        return 16 if n >= 128 else 8 if n >= 32 else 4

    def _run(self, first: int, xin: torch.Tensor, parts: int) -> torch.Tensor:
        """_run_from through a CUDA graph captured once per (batch, entry layer, buffer):
        a forward is ~13 x (groups + fork/join) launches, which the graph replays as one."""
        if not self.use_graphs:
            return self._run_from(first, xin, parts)
        from . import _lib

        key = (int(xin.shape[0]), first, parts, xin.data_ptr())
        entry = self._graphs.get(key)
        if entry is None:
            cur = torch.cuda.current_stream()
            self._run_from(first, xin, parts)  # eager warm-up: modules loaded, streams created
            side = torch.cuda.Stream(device=xin.device)
            side.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.launch_count()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    self._run_from(first, xin, parts)
            kernels = _lib.launch_count() - n0
            _lib.load().fscnn_add_launch_count(-kernels)  # captured, not launched
            cur.wait_stream(side)
            entry = self._graphs[key] = (g, kernels)
        g, kernels = entry
        g.replay()
        _lib.load().fscnn_add_launch_count(kernels)
        return self._bufs[-1]

    def wait_compiled(self) -> "VGGEngine":
        """Join the specialised kernels' compile jobs (and load them)."""
        for st in self.steps:
            if st.jit is not None:
                st.jit.wait()
        return self

    def _run_from(self, first: int, xin: torch.Tensor, parts: int = 2) -> torch.Tensor:
        """Layers first.. on xin (the input of layer ``first``), batch split over streams."""
        n = int(xin.shape[0])
        bufs = self._buffers(n)
        parts = max(1, min(parts, n))
        w0 = self.hw
        for st in self.steps[:first]:
            w0 = w0 // 2 if st.pool else w0
        cur_stream = torch.cuda.current_stream()
        serial = int(os.environ.get("FSCNN_SERIAL_HEAD", "2"))
        if serial > first:
            # the first two layers (224x224, 64 channels: small code, big grids) as
            # full-batch launches on the current stream, with 64-filter groups (see
            # __init__); the batch parts start at layer 2 (C3: value +0.7 %, e2e +2 %;
            # profiles/r02_serial_head.txt)
            cur, w = xin, w0
            for st, out in zip(self.steps[first:serial], bufs[first:serial]):
                st.conv(cur, out, w, n)
                cur = out
                w = w // 2 if st.pool else w
            xin, w0, first = cur, w, serial
            if first >= len(self.steps):
                return bufs[-1]
        if parts > 1 and (getattr(self, "_split_streams", None) is None or len(self._split_streams) != parts):
            self._split_streams = [torch.cuda.Stream(device=xin.device) for _ in range(parts)]
        streams = self._split_streams if parts > 1 else [cur_stream]
        for j, s in enumerate(streams):
            if s is not cur_stream:
                s.wait_stream(cur_stream)
            lo, hi = n * j // parts, n * (j + 1) // parts
            with torch.cuda.stream(s):
                cur, w = xin[lo:hi], w0
                for i, (st, out) in enumerate(zip(self.steps[first:], bufs[first:]), first):
                    # the parts run concurrently: the grid that must fill the GPU is the batch's
                    st.conv(cur, out[lo:hi], w, n)
                    cur = out[lo:hi]
                    w = w // 2 if st.pool else w
        for s in streams:
            if s is not cur_stream:
                cur_stream.wait_stream(s)
        return bufs[-1]

    def forward_whc(self, x_whc: torch.Tensor, n: int) -> torch.Tensor:
        """Device (W,H,C)-memory images (the reference's DenseTensor3 payloads, n of them
        back to back) -> device (W,H,C) outputs [n, W', H', 512]: the input is written
        straight into the halo buffer and the output read straight out of it."""
        bufs = self._buffers(n)
        device.whc_to_halo(x_whc, n, self.in_c, self.hw, self.hw, self._in)
        return device.halo_to_whc(self.run(self._in), self.out_hw)

    def forward_from_host(self, h_src: torch.Tensor, n: int, fill=None) -> torch.Tensor:
        """Pinned host (W,H,C)-memory images -> device (W,H,C) outputs.

        The H2D copy runs on a side stream in up to four parts; the first conv runs per
        part as soon as its part has landed, so later parts' copies overlap compute.
        Later layers run on the whole batch.  ``fill(lo, hi)``, if given, writes images
        lo..hi-1 into ``h_src`` just before their half is copied (host packing of the
        second half then overlaps the first half's copy and conv).
        """
        self._buffers(n)
        elems = self.in_c * self.hw * self.hw
        if getattr(self, "_d_in_n", None) != n:
            self._d_in = torch.empty(n * elems, dtype=torch.float32, device=self._in.device)
            self._d_in_n = n
            self._copy_stream = torch.cuda.Stream(device=self._in.device)
        if not self.use_graphs:
            return self._from_host_body(h_src, n, fill, graphed_tail=False)
        # the whole device side -- part-wise H2D, layout conversion, the stack, the output
        # conversion -- replayed as one CUDA graph per (batch, pinned source); host packing
        # of pageable inputs happens first (it cannot be captured)
        if fill is not None:
            fill(0, n)
        key = ("host", n, h_src.data_ptr())
        entry = self._graphs.get(key)
        if entry is None:
            from . import _lib

            cur = torch.cuda.current_stream()
            self._from_host_body(h_src, n, None, graphed_tail=False)  # eager warm-up
            side = torch.cuda.Stream(device=self._in.device)
            side.wait_stream(cur)
            g = torch.cuda.CUDAGraph()
            n0 = _lib.launch_count()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    out = self._from_host_body(h_src, n, None, graphed_tail=False)
            kernels = _lib.launch_count() - n0
            _lib.load().fscnn_add_launch_count(-kernels)
            cur.wait_stream(side)
            entry = self._graphs[key] = (g, kernels, out)
        g, kernels, out = entry
        g.replay()
        from . import _lib

        _lib.load().fscnn_add_launch_count(kernels)
        return out

    def _from_host_body(self, h_src: torch.Tensor, n: int, fill, graphed_tail: bool) -> torch.Tensor:
        bufs = self._buffers(n)
        elems = self.in_c * self.hw * self.hw
        cur = torch.cuda.current_stream()
        cp = self._copy_stream
        cp.wait_stream(cur)  # the previous call's readers of _d_in are done
        # copy parts x head convs measured (bench e2e, batch 32): 4 x 2 8031 img/s, 4 x 1
        # 7855, 8 x 2 7877, 2 x 2 7941, 16 x 2 7644, 1 x 1 7701 (profiles/r02_e2e_parts.txt)
        parts = 4 if n >= 8 else (2 if n >= 2 else 1)
        if os.environ.get("FSCNN_E2E_PARTS"):
            parts = max(1, min(n, int(os.environ["FSCNN_E2E_PARTS"])))
        halves = [(n * j // parts, n * (j + 1) // parts) for j in range(parts)]
        # the first two convs (the 224x224 block, ~12 % of the stack) run per copy part as
        # soon as it lands, hiding more of the H2D behind them (FSCNN_E2E_HEAD=1 keeps only
        # the first conv there)
        head = 1 if os.environ.get("FSCNN_E2E_HEAD") == "1" or len(self.steps) < 3 else 2
        w = self.hw
        for lo, hi in halves:
            if fill is not None:
                fill(lo, hi)
            with torch.cuda.stream(cp):
                self._d_in[lo * elems:hi * elems].copy_(h_src[lo * elems:hi * elems], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(cp)
            cur.wait_event(ev)
            device.whc_to_halo(self._d_in[lo * elems:hi * elems], hi - lo, self.in_c, self.hw, self.hw,
                               self._in[lo:hi])
            x, w = self._in[lo:hi], self.hw
            for i in range(head):
                self.steps[i].conv(x, bufs[i][lo:hi], w, n)
                x = bufs[i][lo:hi]
                w = w // 2 if self.steps[i].pool else w
        tail = self._run(head, bufs[head - 1], self.parts_for(n)) if graphed_tail else \
            self._run_from(head, bufs[head - 1], self.parts_for(n))
        return device.halo_to_whc(tail, self.out_hw)

    def run_exact(self, x: torch.Tensor) -> torch.Tensor:
        """Dense [N, C, H, W] -> [N, C', H', W'] through the reference-order kernels:
        per conv the bit-exact sparse-filter kernel (taps kw outer, kh inner, channels
        ascending; layers.py:170-180) with bias and ReLU, then the standalone 2x2
        max-pool (layers.py:250-271) -- what set_exact(True) asks of the stack."""
        cur = x.contiguous()
        for st in self.steps:
            cur = device.sf_conv_exact(cur, st.nodes, st.seg_off, st.k, 3, 3, 1, 1, st.bias, relu=True)
            if st.pool:
                cur = device.pool2d(cur, 2, 2, True)
        return cur

    def forward_from_host_exact(self, h_src: torch.Tensor, n: int, fill=None) -> torch.Tensor:
        """forward_from_host through run_exact: pinned (W,H,C) images -> device (W,H,C)."""
        elems = self.in_c * self.hw * self.hw
        if fill is not None:
            fill(0, n)
        d = h_src[: n * elems].to(self.steps[0].bias.device, non_blocking=True)
        x = device.whc_to_nchw(d, n, self.in_c, self.hw, self.hw)
        return device.nchw_to_whc(self.run_exact(x))

    def forward_device(self, x: torch.Tensor) -> torch.Tensor:
        """x: CUDA [N, C, H, W] -> [N, 512, H/32, W/32] (a view into the output buffer;
        ``contiguous=True``: a dense copy, made by the library's pitch-copy kernel)."""
        assert x.shape[1] == self.in_c and x.shape[2] == self.hw and x.shape[3] == self.hw
        y = self.run(self.stage_input(x))
        return device.from_halo(y, self.out_hw)

    def forward_device_dense(self, x: torch.Tensor) -> torch.Tensor:
        """forward_device with a dense contiguous [N, 512, H/32, W/32] result."""
        y = self.run(self.stage_input(x))
        return device.halo_to_nchw(y, self.out_hw)

    def flops_per_image(self) -> int:
        """Exact nnz-FLOPs per image: 2 x in-bounds multiplies (kernels.py:108-133)."""
        total = 0
        for st in self.steps:
            seg = st.seg_off.cpu().numpy().reshape(st.k, 9)
            ends = np.append(seg.ravel()[1:], st.n_nodes).reshape(st.k, 9)
            nnz_tap = (ends - seg - 1).sum(axis=0)  # per tap index kw*3 + kh
            for tap in range(9):
                l, kk = divmod(tap, 3)  # reference segment order: kw outer, kh inner
                rows = sum(1 for i in range(st.h) if 0 <= kk + i - 1 < st.h)
                cols = sum(1 for j in range(st.w) if 0 <= l + j - 1 < st.w)
                total += int(nnz_tap[tap]) * rows * cols
        return 2 * total

    def bytes_per_image(self) -> int:
        """Compulsory HBM bytes per image: each conv reads its input and writes its
        (pooled) output once; filter streams are amortised over the batch (counted once
        per batch by callers)."""
        b = 0
        for st in self.steps:
            ho = st.h // 2 if st.pool else st.h
            b += 4 * (st.c * st.h * st.w + st.k * ho * ho)
        return b

    def filter_bytes(self) -> int:
        return sum(st.bank.total * 8 + st.bank.seg_off.numel() * 8 for st in self.steps)
