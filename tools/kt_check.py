"""The fast sparse-filter kernel with 2, 4 and 8 filters per warp: bit-identical outputs
(each filter's accumulation order does not depend on KT) and the device time of each
VGG16 layer at a given batch.

usage: python tools/kt_check.py [--batch 1] [--zf 0.9] [--layers 0,...,12]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2212_08815_b200 import device, workloads as wl


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--zf", type=float, default=0.9)
    ap.add_argument("--layers", default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    shapes = wl.vgg16_conv_shapes()
    layers = [int(v) for v in args.layers.split(",")] if args.layers else range(len(shapes))
    for li in layers:
        c, k, h, w = shapes[li]
        x, wt, b = wl.sweep_layer(li, "sf", args.zf, n=args.batch)
        xh = device.to_halo(torch.from_numpy(x).cuda())
        bias = torch.from_numpy(b).cuda()
        wd = torch.from_numpy(wt).cuda()
        res, outs = [], []
        for kt, cw in ((4, 0), (2, 0), (8, 0), (2, 4), (1, 0)):
            bank = device.sf_pack(wd, kt)
            out = device.halo_empty(args.batch, k, h, w)
            fn = lambda: device.sf_conv3x3(xh, bank, bias, True, False, out=out, w=w, cta_warps=cw)
            fn()
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(args.reps):
                fn()
            e.record()
            e.synchronize()
            res.append((f"{kt}" + ("/4w" if cw or kt == 1 else ""), a.elapsed_time(e) / args.reps * 1e3))
            outs.append(out.clone())
        same = all(torch.equal(outs[0].view(torch.int32), o.view(torch.int32)) for o in outs[1:])
        print(f"L{li} {c}->{k} @{h} batch {args.batch}: " + ", ".join(f"kt{kt} {us:.1f} us" for kt, us in res)
              + f"  bit-identical: {same}", flush=True)


if __name__ == "__main__":
    main()
