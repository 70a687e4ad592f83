"""Does the fast SF kernel's speed depend on the input values?  Times one VGG16 layer
with N(0,1) input, all-zero input and a constant input (same filter bank)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_08815_b200 import device, workloads as wl

li = int(sys.argv[1]) if len(sys.argv) > 1 else 5
c, k, h, w = wl.vgg16_conv_shapes()[li]
x, wt, b = wl.sweep_layer(li, "sf", 0.9, n=32)
bank = device.sf_pack(torch.from_numpy(wt).cuda())
bias = torch.from_numpy(b).cuda()
out = device.halo_empty(32, k, h, w)
xr = torch.from_numpy(x).cuda()
for name, xx in (("normal", xr), ("zeros", torch.zeros_like(xr)), ("ones", torch.ones_like(xr)),
                 ("normal", xr)):
    xh = device.to_halo(xx)
    for _ in range(3):
        device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, out=out)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        device.sf_conv3x3(xh, bank, bias, relu=True, pool=False, w=w, out=out)
    e.record(); e.synchronize()
    print(f"L{li} {name:7s} {a.elapsed_time(e) / 10:.3f} ms", flush=True)
