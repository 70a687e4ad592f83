"""Run one VGG16 layer's sparse-input conv (batch 32) for profiling / timing.

usage: python tools/prof_si.py LAYER [ZERO_FRAC] [REPS] [exact|fast]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_08815_b200 import device, workloads as wl

li = int(sys.argv[1]) if len(sys.argv) > 1 else 8
zf = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
mode = sys.argv[4] if len(sys.argv) > 4 else "exact"
c, k, h, w = wl.vgg16_conv_shapes()[li]
x, wt, b = wl.sweep_layer(li, "si", zf, n=32)
xd = torch.from_numpy(x).cuda()
enc = device.encode_order(xd, "CHW")
out = torch.empty((32, k, h, w), dtype=torch.float32, device="cuda")
if mode == "fast":
    wf = device.si_pack_fast(torch.from_numpy(wt).cuda())
    run = lambda: device.si_conv3x3_fast(enc.nodes, enc.seg_off, 32, c, h, w, wf, k, out=out)
else:
    wq = device.si_pack3x3(torch.from_numpy(wt).cuda())
    run = lambda: device.si_conv3x3(enc.nodes, enc.seg_off, 32, c, h, w, wq, k, out=out)
for _ in range(2):
    run()
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(reps):
    run()
e.record(); e.synchronize()
ms = a.elapsed_time(e) / reps
nz = x != 0
rows = np.array([sum(1 for kh in range(3) if 0 <= i + 1 - kh < h) for i in range(h)])
cols = np.array([sum(1 for kw in range(3) if 0 <= j + 1 - kw < w) for j in range(w)])
fl = 2 * k * int((nz * (rows[:, None] * cols[None, :])[None, None]).sum())
print(f"SI ({mode}) layer {li} {(c, k, h, w)} zf {zf}: {ms:.3f} ms  {fl / ms / 1e9:.2f} TFLOP/s", flush=True)
