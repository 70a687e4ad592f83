"""BASELINE config 2's sparse-input kernel, a few calls (for ncu): python tools/prof_c2.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402

x, wt, b = wl.c2()
xd = torch.from_numpy(x).cuda()
wq = device.si_pack3x3(torch.from_numpy(wt).cuda())
enc = device.encode_order(xd, "CHW")
y = torch.empty((1, 128, 28, 28), dtype=torch.float32, device="cuda")
for _ in range(3):
    device.si_conv3x3(enc.nodes, enc.seg_off, 1, 128, 28, 28, wq, 128, out=y)
torch.cuda.synchronize()
print("ok")
