"""torch.profiler view of one batched network.forward (kernel device time vs wall clock).

usage: python tools/prof_variant.py [--variant sparse_input] [--batch 32] [--density 0.5]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

import paper_2212_08815_b200 as fs
from paper_2212_08815_b200 import network as nw

ap = argparse.ArgumentParser()
ap.add_argument("--variant", default="sparse_input")
ap.add_argument("--batch", type=int, default=32)
ap.add_argument("--density", type=float, default=0.5)
args = ap.parse_args()
net = nw.build_benchmark_net("vgg16_desk", 1.0, input_hw=224, variant=args.variant)
prepared = nw.prepare(net, nw.random_weights(net, 7))
xs = [fs.prune_random(nw.random_input(net.input_dims, 100 + i), args.density, 100 + i) for i in range(args.batch)]
inp = [fs.sparsify_tensor3(x, fs.AxisOrder3.CHW) if args.variant == "sparse_input" else x for x in xs]
nw.forward(prepared, inp)
torch.cuda.synchronize()
t0 = time.perf_counter()
nw.forward(prepared, inp)
print(f"wall {1e3 * (time.perf_counter() - t0):.1f} ms")
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CPU, torch.profiler.ProfilerActivity.CUDA]) as p:
    nw.forward(prepared, inp)
    torch.cuda.synchronize()
print(p.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
print(p.key_averages().table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=60))
import cProfile
import pstats

pr = cProfile.Profile()
pr.enable()
nw.forward(prepared, inp)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
