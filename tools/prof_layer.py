"""Run one VGG16 layer's fast sparse-filter conv (batch 32, 90% zeros) for profiling.

usage: python tools/prof_layer.py LAYER [REPS]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_08815_b200 import device, workloads as wl

li = int(sys.argv[1]) if len(sys.argv) > 1 else 1
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c, k, h, w = wl.vgg16_conv_shapes()[li]
x, wt, b = wl.sweep_layer(li, "sf", 0.9, n=32)
bank = device.sf_pack(torch.from_numpy(wt).cuda())
xh = device.to_halo(torch.from_numpy(x).cuda())
bias = torch.from_numpy(b).cuda()
ly = device.pick_ly(c, h)
print("layer", li, (c, k, h, w), "ly", ly, "plan", bank.chunk_plan(ly), flush=True)
for _ in range(reps):
    y = device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, ly=ly)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
y = device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, ly=ly)
e.record(); e.synchronize()
ms = a.elapsed_time(e)
flops = 2 * bank.nnz * h * w * 32  # approx (ignores border taps)
print(f"ms {ms:.3f}  approx TFLOP/s {flops / ms / 1e9:.2f}", flush=True)
