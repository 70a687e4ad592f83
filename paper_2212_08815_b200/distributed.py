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


def max_over_ranks(value: float, device, group=None) -> float:
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
