"""Batch-sharded multi-GPU driver for the VGG16 sparse-filter stack.

One process per GPU (torchrun), torch.distributed over NCCL.  The path shards on the
batch: every image is independent (the reference's instance-parallel mode,
network.py:498-515), so there is no per-layer exchange.  Communication happens
exactly twice, as the north star prescribes:

  1. once per weight set, rank 0's encoded filter banks (reference CHW node format:
     nodes + segment/matrix/tensor offsets + bias) are broadcast to all ranks; each
     rank derives its kernel-side packed stream locally from the received nodes;
  2. the final activations of every shard are gathered (rank order) at the end.

Determinism: a rank computes exactly what a single GPU computes for the same images
(the kernels are batch-position invariant), so 1/2/4/8-GPU outputs are byte-identical.
The helpers are device-agnostic (gloo + CPU tensors in the unit tests, NCCL + CUDA
tensors on the box).
"""

from __future__ import annotations

import time

import numpy as np
import torch
import torch.distributed as dist


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous slice [lo, hi) of ``total`` items for ``rank`` (remainder to low ranks)."""
    base, extra = divmod(total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def broadcast_banks(banks, device, src: int = 0, group=None):
    """Broadcast encoded banks from ``src``.

    banks (on src): list of tuples (nodes int32 [n, 2], seg_off int64, tensor_off int64,
    matrix_off int64, bias float32) -- other ranks pass None.
    Returns the same list (tensors on ``device``) on every rank.
    """
    rank = dist.get_rank(group)
    if rank == src:
        n_layers = torch.tensor([len(banks)], dtype=torch.int64, device=device)
    else:
        n_layers = torch.zeros(1, dtype=torch.int64, device=device)
    dist.broadcast(n_layers, src, group=group)
    out = []
    for i in range(int(n_layers.item())):
        if rank == src:
            parts = [t.to(device).contiguous() for t in banks[i]]
            hdr = torch.tensor([p.numel() for p in parts], dtype=torch.int64, device=device)
        else:
            hdr = torch.zeros(5, dtype=torch.int64, device=device)
        dist.broadcast(hdr, src, group=group)
        if rank != src:
            sizes = [int(v) for v in hdr.tolist()]
            parts = [
                torch.empty((sizes[0] // 2, 2), dtype=torch.int32, device=device),
                torch.empty(sizes[1], dtype=torch.int64, device=device),
                torch.empty(sizes[2], dtype=torch.int64, device=device),
                torch.empty(sizes[3], dtype=torch.int64, device=device),
                torch.empty(sizes[4], dtype=torch.float32, device=device),
            ]
        for p in parts:
            dist.broadcast(p, src, group=group)
        out.append(tuple(parts))
    return out


def gather_outputs(y: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather equally shaped per-rank output shards (rank order)."""
    world = dist.get_world_size(group)
    bufs = [torch.empty_like(y) for _ in range(world)]
    dist.all_gather(bufs, y.contiguous(), group=group)
    return bufs


def comm_device(device: torch.device, group=None) -> torch.device:
    """Where collective buffers live: the GPU under NCCL, host memory under gloo (the
    CPU tests, and one-GPU multi-process tests that cannot run NCCL on a shared GPU)."""
    return device if dist.get_backend(group) == "nccl" else torch.device("cpu")


def gather_batch(y_local: torch.Tensor, total: int, group=None, out: torch.Tensor | None = None) -> torch.Tensor:
    """Rank-ordered all-gather of per-rank batch shards [n_r, ...] (n_r from shard_range,
    possibly unequal) into the full [total, ...] batch on every rank.

    Equal shards on the collective's own device (NCCL, total % world == 0 -- every bench
    configuration) are ONE collective straight into ``out`` (or a fresh tensor): no
    padding, no staging copies, no concatenation.  Unequal shards are padded to the
    largest one and trimmed after the gather."""
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(total, rank, world)
    assert int(y_local.shape[0]) == hi - lo
    if total % world == 0 and comm_device(y_local.device, group) == y_local.device and y_local.is_contiguous():
        shape = (total,) + tuple(y_local.shape[1:])
        if out is None or tuple(out.shape) != shape or out.dtype != y_local.dtype or out.device != y_local.device:
            out = torch.empty(shape, dtype=y_local.dtype, device=y_local.device)
        dist.all_gather_into_tensor(out, y_local, group=group)
        return out
    n_max = shard_range(total, 0, world)[1]  # rank 0 holds the largest shard
    dev = comm_device(y_local.device, group)
    pad = torch.zeros((n_max,) + tuple(y_local.shape[1:]), dtype=y_local.dtype, device=dev)
    pad[: hi - lo].copy_(y_local)
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    parts = []
    for r in range(world):
        a, b = shard_range(total, r, world)
        parts.append(bufs[r][: b - a])
    return torch.cat(parts).to(y_local.device)


def max_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class ShardedVGG:
    """Batch-sharded VGG16 sparse-filter stack: one process (one GPU) per rank.

    Construction (collective): rank 0 encodes every filter bank on its GPU into the
    reference CHW node format; the banks are broadcast once (broadcast_banks) and every
    rank builds its own engine from them (the packed kernel streams are derived
    locally).  ``forward`` is the SPMD counterpart of network.forward
    (network.py:478-534, instance-parallel over workers at :498-515): every rank passes
    the same full batch, runs its contiguous shard (shard_range) through the engine, and
    the device outputs are all-gathered in rank order before one D2H -- so every rank
    returns the full output list, byte-identical to a single-GPU forward (the kernels
    are batch-position invariant; tests/test_gpu_api.py::test_sharded_forward_*).
    """

    def __init__(self, layers, hw: int = 224, group=None, device: torch.device | None = None,
                 plan=None, in_c: int = 3):
        from .engine import VGGEngine
        from .workloads import VGG16_PLAN

        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        plan = list(plan or VGG16_PLAN)
        cdev = comm_device(self.device, group)
        if self.rank == 0:
            eng0 = VGGEngine(layers, batch=1, hw=hw, plan=plan, in_c=in_c)
            if self.world > 1:
                # rank 0 compiles the specialised kernels alone while the other ranks wait
                # in the broadcast; they then find every cubin in the shared disk cache
                # (same PTX on every rank) instead of all ranks compiling the same code
                eng0.wait_compiled()
            banks = [(s.nodes[: s.n_nodes], s.seg_off, s.tensor_off, s.matrix_off, s.bias) for s in eng0.steps]
            banks = [tuple(t.to(cdev) for t in b) for b in banks]
        else:
            banks = None
        got = broadcast_banks(banks, cdev, group=group)
        if self.rank == 0:
            self.engine = eng0
        else:
            enc = []
            for nodes, seg, ten, mat, bias in got:
                nodes, seg, ten, mat = (t.to(self.device) for t in (nodes, seg, ten, mat))
                enc.append((nodes, int(nodes.shape[0]), seg, ten, mat, bias.cpu().numpy(), int(ten.numel())))
            self.engine = VGGEngine(None, batch=1, hw=hw, plan=plan, in_c=in_c, encoded=enc)
        from . import network

        self.prepared = network.prepared_from_engine(self.engine)

    def shard(self, total: int) -> tuple[int, int]:
        return shard_range(total, self.rank, self.world)

    def forward_device(self, x: torch.Tensor, total: int | None = None) -> torch.Tensor:
        """This rank's shard x [n_r, C, H, W] (on its GPU) -> the gathered full-batch
        output [total, 512, H/32, W/32] on every rank."""
        total = int(x.shape[0]) * self.world if total is None else total
        y = self.engine.forward_device_dense(x)
        # equal shards gather into one reused buffer (valid until the next call, like the
        # engine's own output buffers)
        self._full = gather_batch(y, total, self.group, out=getattr(self, "_full", None))
        return self._full

    def forward(self, batch: list, dst: int | None = None) -> list | None:
        """network.forward for the batch-sharded stack: host DenseTensor3 list in (the same
        full list on every rank), host DenseTensor3 list out -- on every rank, or only on
        rank ``dst`` (the others return None and skip the D2H)."""
        from . import network

        network._check_batch(self.prepared, batch)
        n = len(batch)
        lo, hi = self.shard(n)
        eng = self.engine
        with network._engine_lock:
            if hi > lo:
                whc = network._engine_device_forward(self.prepared, batch[lo:hi])
            else:
                whc = torch.empty((0, eng.out_hw, eng.out_hw, eng.out_c), dtype=torch.float32, device=self.device)
            full = gather_batch(whc, n, self.group)
            if dst is not None and dst != self.rank:
                torch.cuda.current_stream().synchronize()
                return None
            return network._whc_to_host(full, n, eng.out_c, eng.out_hw)

    def timed_forward(self, batch: list, dst: int | None = None, reps: int = 1) -> tuple[list, float]:
        """``reps`` forwards after a barrier; returns (last outputs, seconds) with the seconds
        the max over ranks of each rank's wall clock (the multi-GPU e2e timing rule)."""
        dist.barrier(self.group)
        t0 = time.perf_counter()
        for _ in range(reps):
            out = self.forward(batch, dst)
        dt = time.perf_counter() - t0
        return out, max_over_ranks(dt, comm_device(self.device, self.group), self.group)
