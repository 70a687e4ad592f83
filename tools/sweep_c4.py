"""BASELINE config 4: per-layer sparsity sweep on the 13 VGG16 conv shapes at batch 32.

Sparse-filter conv (fused ReLU, no pool) at filter sparsity {50,75,90,95,99}%: the
specialised per-layer kernels ("sf", sfjit.cu) and the jump-table kernel ("sf_jt",
sf3x3_kernel), each with its normwise error against the reference-order exact kernel
(pinned bit-exact to the reference) on the first 2 images.  Sparse-input conv at input
sparsity {50,75,90,95}% on the device-encoded input: the bit-exact strip kernel ("si")
and the channel-major kernel ("si_fast", normwise error against "si").

Each point: device time from CUDA events (median of reps), exact nnz-FLOPs, achieved
TFLOP/s, and the north-star roofline: t_roof = max(nnz-FLOPs / FP32 peak, compulsory
bytes / HBM bandwidth), frac = t_roof / t_measured, bound = whichever term is larger.
Compulsory bytes: SF -- input + output activations (fp32) + the filter nodes (8 B
each); SI -- input nodes (8 B each) + segment offsets + dense filters + output.
Writes JSON lines to stdout (one per point) and, with --out, a JSON file.

usage: python tools/sweep_c4.py [--out profiles/r01_c4_sweep.json] [--layers 0,1,...] [--reps 5]
       [--modes sf,si,si_fast]
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


def time_fn(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def sf_flops(wt, h, w, n):
    """2 x exact in-bounds multiplies for 3x3/s1/p1 (kernels.py:108-133)."""
    k, c = wt.shape[:2]
    total = 0
    for kh in range(3):
        rows = sum(1 for i in range(h) if 0 <= kh + i - 1 < h)
        for kw in range(3):
            cols = sum(1 for j in range(w) if 0 <= kw + j - 1 < w)
            total += int(np.count_nonzero(wt[:, :, kh, kw])) * rows * cols
    return 2 * total * n


def si_flops(x, k):
    """2 x K x sum over input nonzeros of their in-bounds taps."""
    n, c, h, w = x.shape
    nz = x != 0
    rows = np.array([sum(1 for kh in range(3) if 0 <= i + 1 - kh < h) for i in range(h)])
    cols = np.array([sum(1 for kw in range(3) if 0 <= j + 1 - kw < w) for j in range(w)])
    taps = rows[:, None] * cols[None, :]
    return 2 * k * int((nz * taps[None, None]).sum())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--layers", default=None)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--peak", type=float, default=72.3, help="FP32 TFLOP/s denominator (measured probe)")
    ap.add_argument("--hbm", type=float, default=None, help="HBM GB/s (default MEASURED_PEAKS.json)")
    ap.add_argument("--modes", default="sf,sf_jt,si,si_fast")
    ap.add_argument("--zf", default=None, help="comma list restricting the zero fractions")
    args = ap.parse_args()
    if args.hbm is None:
        try:
            root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
            args.hbm = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
        except (OSError, KeyError, ValueError):
            args.hbm = 6460.9

    def roof(r, nbytes):
        t_flop = r["nnz_gflop"] / args.peak          # ms (GFLOP / TFLOP/s)
        t_hbm = nbytes / 1e9 / args.hbm * 1e3        # ms
        r["bytes"] = int(nbytes)
        r["roofline_ms"] = max(t_flop, t_hbm)
        r["bound"] = "fp32" if t_flop >= t_hbm else "hbm"
        r["frac"] = r["roofline_ms"] / r["ms"]
        r["frac_of_fp32_peak"] = r["tflops"] / args.peak
        return r

    def zfs(default):
        return [float(v) for v in args.zf.split(",")] if args.zf else default

    shapes = wl.vgg16_conv_shapes()
    layers = [int(v) for v in args.layers.split(",")] if args.layers else range(len(shapes))
    rows = []
    for li in layers:
        c, k, h, w = shapes[li]
        modes = args.modes.split(",")
        for zf in zfs((0.5, 0.75, 0.9, 0.95, 0.99)) if ("sf" in modes or "sf_jt" in modes) else ():
            x, wt, b = wl.sweep_layer(li, "sf", zf, n=args.n)
            wd = torch.from_numpy(wt).cuda()
            xh = device.to_halo(torch.from_numpy(x).cuda())
            bias = torch.from_numpy(b).cuda()
            out = device.halo_empty(args.n, k, h, w)
            fl = sf_flops(wt, h, w, args.n)
            nnz = int(np.count_nonzero(wt))
            nbytes = 4 * args.n * (c + k) * h * w + 8 * nnz
            # parity: the exact kernel (bit-exact with the reference) on the first 2 images
            enc = device.encode_order(wd, "CHW")
            x2 = torch.from_numpy(x[:2]).cuda()
            ex = device.sf_conv_exact(x2, enc.nodes, enc.seg_off, k, 3, 3, 1, 1, bias, relu=True)
            for mode in ("sf", "sf_jt"):
                if mode not in modes:
                    continue
                if mode == "sf":
                    jit = device.SfJit(wt, b, h, w, relu=True, pool=False).wait()
                    fn = lambda: jit(xh, out=out)
                else:
                    bank = device.sf_pack(wd)
                    fn = lambda: device.sf_conv3x3(xh, bank, bias, True, False, out=out, w=w)
                ms = time_fn(fn, args.reps)
                got = device.from_halo(out, w)[:2]
                err = float((got - ex).abs().max() / ex.abs().max().clamp_min(1e-30))
                r = {"mode": mode, "layer": li, "shape": [c, k, h, w], "zero_frac": zf, "ms": ms,
                     "nnz_gflop": fl / 1e9, "tflops": fl / (ms * 1e-3) / 1e12,
                     "normwise_err_vs_exact": err}
                rows.append(roof(r, nbytes))
                print(json.dumps(r), flush=True)
            del xh, out, enc, x2, ex
        for zf in zfs((0.5, 0.75, 0.9, 0.95)) if ("si" in modes or "si_fast" in modes) else ():
            x, wt, b = wl.sweep_layer(li, "si", zf, n=args.n)
            xd = torch.from_numpy(x).cuda()
            enc = device.encode_order(xd, "CHW")
            fl = si_flops(x, k)
            nbytes = 8 * int(enc.n_nodes) + 8 * int(enc.seg_off.numel()) + 4 * k * c * 9 + 4 * args.n * k * h * w
            ref = None
            for mode in ("si", "si_fast"):
                if mode not in modes:
                    continue
                out = torch.empty((args.n, k, h, w), dtype=torch.float32, device="cuda")
                if mode == "si":
                    wq = device.si_pack3x3(torch.from_numpy(wt).cuda())
                    fn = lambda: device.si_conv3x3(enc.nodes, enc.seg_off, args.n, c, h, w, wq, k, out=out)
                else:
                    wf = device.si_pack_fast(torch.from_numpy(wt).cuda())
                    fn = lambda: device.si_conv3x3_fast(enc.nodes, enc.seg_off, args.n, c, h, w, wf, k, out=out)
                ms = time_fn(fn, args.reps)
                r = {"mode": mode, "layer": li, "shape": [c, k, h, w], "zero_frac": zf, "ms": ms,
                     "nnz_gflop": fl / 1e9, "tflops": fl / (ms * 1e-3) / 1e12}
                roof(r, nbytes)
                if mode == "si":
                    ref = out
                elif ref is not None:  # normwise error of the reassociated sum vs the exact kernel
                    r["normwise_err_vs_exact"] = float((out - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
                rows.append(r)
                print(json.dumps(r), flush=True)
            del xd, enc, out, ref
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(rows, fh, indent=0)


if __name__ == "__main__":
    main()
