"""Time the VGG16 stack (BASELINE config 3 / 5 shapes) for different numbers of
batch-split streams in VGGEngine.run (parts) -- the stream-overlap knob.

usage: python tools/parts_sweep.py [--batch 32] [--zf 0.9] [--parts 1,2,3,4]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_2212_08815_b200 import workloads as wl
from paper_2212_08815_b200.engine import VGGEngine


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--zf", type=float, default=0.9)
    ap.add_argument("--parts", default="1,2,3,4")
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=args.zf), batch=args.batch, hw=224)
    x = torch.from_numpy(wl.vgg16_input(args.batch, seed=104)).cuda()
    xh = eng.stage_input(x)
    for parts in (int(v) for v in args.parts.split(",")):
        for _ in range(3):
            eng.run(xh, parts=parts)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            eng.run(xh, parts=parts)
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / args.reps
        print(f"batch {args.batch} zf {args.zf} parts {parts}: {ms:.3f} ms/step  {args.batch / ms * 1e3:.0f} img/s")


if __name__ == "__main__":
    main()
