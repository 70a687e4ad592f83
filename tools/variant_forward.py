"""Time network.forward for the dense_baseline and sparse_input variants: the batched
device path (one launch per layer for the whole batch, activations in HBM) against the
per-image layer path (network._BATCHED = False), and check they agree bit for bit.
Wall clock per forward call (batched: best of 3).

usage: python tools/variant_forward.py [--kind vgg16_desk] [--scale 1.0] [--hw 224] [--batch 8]
       [--variants sparse_input,dense_baseline,sparse_filter] [--filter-density 0.1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import network as nw


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kind", default="vgg16_desk")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--hw", type=int, default=224)
    ap.add_argument("--batch", type=int, default=8)
    ap.add_argument("--density", type=float, default=0.5)
    ap.add_argument("--variants", default="sparse_input,dense_baseline")
    ap.add_argument("--filter-density", type=float, default=0.1, help="sparse_filter weights kept")
    args = ap.parse_args()
    for variant in args.variants.split(","):
        net = nw.build_benchmark_net(args.kind, args.scale, input_hw=args.hw, variant=variant)
        weights = nw.random_weights(net, 7)
        if variant == "sparse_filter":
            weights = nw.prune_weights(weights, args.filter_density, 7)
        prepared = nw.prepare(net, weights)
        xs = [fs.prune_random(nw.random_input(net.input_dims, 100 + i), args.density, 100 + i)
              for i in range(args.batch)]
        inp = [fs.sparsify_tensor3(x, fs.AxisOrder3.CHW) if variant == "sparse_input" else x for x in xs]
        def best(reps=3):
            t, out = 1e30, None
            for _ in range(reps):
                t0 = time.perf_counter()
                out = nw.forward(prepared, inp).outputs
                t = min(t, time.perf_counter() - t0)
            return t, out

        nw.forward(prepared, inp)  # warm-up (allocations, library load)
        t_b, a = best()
        nw._BATCHED = False
        t_s, b = best(1)
        nw._BATCHED = True
        same = all((x.nodes.tobytes() == y.nodes.tobytes()) if isinstance(x, fs.SparseTensor3)
                   else np.array_equal(np.asarray(x.data).view(np.int32), np.asarray(y.data).view(np.int32))
                   for x, y in zip(a, b))
        print(f"{args.kind} x{args.scale} @{args.hw} {variant} batch {args.batch}: batched {t_b * 1e3:.1f} ms "
              f"({args.batch / t_b:.1f} img/s), per-image {t_s * 1e3:.1f} ms ({args.batch / t_s:.1f} img/s), "
              f"identical: {same}", flush=True)


if __name__ == "__main__":
    main()
