"""Time the fast sparse-filter kernel on all 13 VGG16 layer shapes (batch 32).

usage: python tools/layer_sweep.py [ZERO_FRAC] [REPS]   -> one line per layer + total
       SWEEP_LY=2|4|8 forces the sub-region height; SWEEP_LAYERS=1,5 selects layers
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_08815_b200 import device, workloads as wl

zf = float(sys.argv[1]) if len(sys.argv) > 1 else 0.9
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tot_ms = tot_fl = 0.0
only = os.environ.get("SWEEP_LAYERS")
for li, (c, k, h, w) in enumerate(wl.vgg16_conv_shapes()):
    if only and str(li) not in only.split(","):
        continue
    x, wt, b = wl.sweep_layer(li, "sf", zf, n=32)
    bank = device.sf_pack(torch.from_numpy(wt).cuda())
    xh = device.to_halo(torch.from_numpy(x).cuda())
    bias = torch.from_numpy(b).cuda()
    ly = int(os.environ.get("SWEEP_LY", "0")) or device.pick_ly(c, h)
    out = device.halo_empty(32, k, h, w)
    for _ in range(2):
        device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, ly=ly, out=out)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, ly=ly, out=out)
    e.record(); e.synchronize()
    ms = a.elapsed_time(e) / reps
    fl = 2.0 * bank.nnz * h * w * 32 * (1 - 2.0 / (3 * h))  # approx border correction
    tot_ms += ms; tot_fl += fl
    print(f"L{li:2d} {c:3d}->{k:3d} @{h:3d} ly{ly} plan{bank.chunk_plan(ly)}  {ms:7.3f} ms  {fl / ms / 1e9:6.2f} TFLOP/s", flush=True)
print(f"total {tot_ms:.3f} ms  {tot_fl / tot_ms / 1e9:.2f} TFLOP/s")
