"""The HBM-bound kernels at VGG16 sizes, for ncu: the encoder (count / scan / write) on a
layer-1 activation in CHW order, the decoder, ReLU, 2x2 max-pool and the WHC <-> NCHW
layout converters.  Prints each kernel's device time and effective GB/s (algorithmic
bytes: read + write once).

usage: python tools/prof_misc.py [--reps 5]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2212_08815_b200 import device


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(1)
    n, c, h, w = 8, 64, 224, 224
    x = torch.randn((n, c, h, w), device="cuda", generator=g)
    x = torch.relu(x)  # ~50 % zeros, like a post-ReLU activation
    elems = x.numel()
    rows = []
    ms = timed(lambda: device.encode_order(x, "CHW"), args.reps)
    enc = device.encode_order(x, "CHW")
    node_bytes = enc.n_nodes * 8 + enc.seg_off.numel() * 8
    rows.append(("encode CHW (count+scan+write, incl. the count sync)", ms, elems * 4 * 2 + node_bytes))
    out = torch.empty_like(x)
    ms = timed(lambda: device.decode_order(enc.nodes, enc.seg_off, (n, c, h, w), "CHW", out=out), args.reps)
    rows.append(("decode CHW", ms, node_bytes + elems * 4))
    y = torch.empty_like(x)
    ms = timed(lambda: device.relu(x, out=y), args.reps)
    rows.append(("relu", ms, elems * 8))
    ms = timed(lambda: device.pool2d(x, 2, 2, True), args.reps)
    rows.append(("maxpool 2x2", ms, elems * 4 + elems))
    whc = device.nchw_to_whc(x)
    ms = timed(lambda: device.nchw_to_whc(x, out=whc), args.reps)
    rows.append(("nchw -> whc", ms, elems * 8))
    ms = timed(lambda: device.whc_to_nchw(whc.view(-1), n, c, h, w, out=y), args.reps)
    rows.append(("whc -> nchw", ms, elems * 8))
    xin = torch.randn((32, 3, 224, 224), device="cuda", generator=g)
    win = device.nchw_to_whc(xin).view(-1)
    hal = device.halo_empty(32, 3, 224, 224)
    ms = timed(lambda: device.whc_to_halo(win, 32, 3, 224, 224, hal), args.reps)
    rows.append(("whc -> halo NCHW, 32 x 3 x 224 x 224 (the network input)", ms, xin.numel() * 8))
    for name, ms, nbytes in rows:
        print(f"{name:55s} {ms * 1e3:9.1f} us  {nbytes / (ms * 1e-3) / 1e9:8.1f} GB/s")


if __name__ == "__main__":
    main()
