"""BASELINE configs 1 and 2 on the GPU (single-image layers; launch-bound by nature).

C1: sparse-filter conv N=1, 64->64 @56x56, 95% filter zeros (workloads.c1): the fast
    kernel on the device-resident halo input, and the reference-order exact kernel.
C2: sparse-input conv N=1, 128->128 @28x28, 90% input zeros (workloads.c2): the GPU
    encoder on the dense input + the strip kernel (and the kernel alone on ready nodes).
Device time per call from CUDA events over many back-to-back calls (median of 5 runs),
plus the same loop captured in a CUDA graph (launch overhead removed).  nnz-FLOPs as
in SURVEY.md §8(d).  Prints one JSON object.

usage: python tools/configs_12.py [--out profiles/r01_configs_12.json]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2212_08815_b200 import device, workloads as wl


def per_call_us(fn, calls=200, runs=5):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(runs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(calls):
            fn()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e3 / calls)
    return statistics.median(out)


def graph_us(fn, calls=200, runs=5):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(calls):
            fn()
    g.replay()
    torch.cuda.synchronize()
    out = []
    for _ in range(runs):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) * 1e3 / calls)
    return statistics.median(out)


def sf_flops(wt, h, w):
    total = 0
    for kh in range(3):
        rows = sum(1 for i in range(h) if 0 <= kh + i - 1 < h)
        for kw in range(3):
            cols = sum(1 for j in range(w) if 0 <= kw + j - 1 < w)
            total += int(np.count_nonzero(wt[:, :, kh, kw])) * rows * cols
    return 2 * total


def si_flops(x, k):
    _, _, h, w = x.shape
    rows = np.array([sum(1 for kh in range(3) if 0 <= i + 1 - kh < h) for i in range(h)])
    cols = np.array([sum(1 for kw in range(3) if 0 <= j + 1 - kw < w) for j in range(w)])
    return 2 * k * int(((x != 0) * (rows[:, None] * cols[None, :])[None, None]).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    res = {}
    # C1
    x, wt, b = wl.c1()
    bank = device.sf_pack(torch.from_numpy(wt).cuda())
    xh = device.to_halo(torch.from_numpy(x).cuda())
    xd = torch.from_numpy(x).cuda()
    bias = torch.from_numpy(b).cuda()
    out = device.halo_empty(1, 64, 56, 56)
    enc = device.encode_order(torch.from_numpy(wt).cuda(), "CHW")
    fl = sf_flops(wt, 56, 56)
    fast = lambda: device.sf_conv3x3(xh, bank, bias, False, False, out=out, w=56)
    kt, warps = device.sf_grid_plan(1, 56, 56, 64, device.pick_ly(64, 56))
    bank_s = device.sf_pack(torch.from_numpy(wt).cuda(), kt)
    fast_small = lambda: device.sf_conv3x3(xh, bank_s, bias, False, False, out=out, w=56, cta_warps=warps)
    exact = lambda: device.sf_conv_exact(xd, enc.nodes, enc.seg_off, 64, 3, 3, 1, 1, bias)
    cases = [("fast", fast), ("fast_small_grid", fast_small), ("exact", exact)]
    for kt in (4, 8, 16, 48):
        j = device.SfJit(wt, b, 56, 56, relu=False, pool=False, flags=kt).wait()
        cases.append((f"sfjit_kt{kt}", (lambda j=j: j(xh, out=out))))
    for kt, wc in ((2, 0), (4, 0), (8, 0), (16, 0), (4, 8), (8, 8), (16, 8)):
        j = device.SfJit(wt, b, 56, 56, relu=False, pool=False, flags=kt | (wc << 8) | (1 << 16)).wait()
        cases.append((f"sfjit_fused_kt{kt}_w{wc}", (lambda j=j: j(xh, out=out))))
    for name, fn in cases:
        us, gus = per_call_us(fn), graph_us(fn)
        res[f"c1_{name}"] = {"us_per_call": us, "us_per_call_graph": gus, "nnz_gflop": fl / 1e9,
                             "nnz_gflops": fl / (gus * 1e-6) / 1e9}
    # C2
    x, wt, b = wl.c2()
    xd = torch.from_numpy(x).cuda()
    wq = device.si_pack3x3(torch.from_numpy(wt).cuda())
    enc = device.encode_order(xd, "CHW")
    y = torch.empty((1, 128, 28, 28), dtype=torch.float32, device="cuda")
    fl = si_flops(x, 128)
    kern = lambda: device.si_conv3x3(enc.nodes, enc.seg_off, 1, 128, 28, 28, wq, 128, out=y)
    us, gus = per_call_us(kern), graph_us(kern)
    res["c2_kernel"] = {"us_per_call": us, "us_per_call_graph": gus, "nnz_gflop": fl / 1e9,
                        "nnz_gflops": fl / (gus * 1e-6) / 1e9}
    wf = device.si_pack_fast(torch.from_numpy(wt).cuda())
    kern_f = lambda: device.si_conv3x3_fast(enc.nodes, enc.seg_off, 1, 128, 28, 28, wf, 128, out=y)
    us, gus = per_call_us(kern_f), graph_us(kern_f)
    res["c2_fast_kernel"] = {"us_per_call": us, "us_per_call_graph": gus, "nnz_gflop": fl / 1e9,
                             "nnz_gflops": fl / (gus * 1e-6) / 1e9,
                             "note": "channel-major kernel (28 CTAs here; the layer API keeps the exact one)"}
    layer = lambda: device.si_conv3x3(*(lambda e: (e.nodes, e.seg_off))(device.encode_order(xd, "CHW")), 1, 128,
                                      28, 28, wq, 128, out=y)
    res["c2_encode_plus_kernel"] = {"us_per_call": per_call_us(layer, calls=50),
                                    "note": "includes the encoder's one host sync (node count)"}
    print(json.dumps(res, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
