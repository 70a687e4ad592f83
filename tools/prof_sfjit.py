"""One layer of the VGG16 stack through sfjit (for ncu): python tools/prof_sfjit.py LAYER [N]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402

li = int(sys.argv[1])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
H = [224, 224, 112, 112, 56, 56, 56, 28, 28, 28, 14, 14, 14][li]
POOL = li in (1, 3, 6, 9, 12)
wt, b = wl.vgg16_weights(seed=103, zero_frac=0.9)[li]
x = device.to_halo(torch.randn(n, wt.shape[1], H, H, device="cuda"))
j = device.SfJit(wt, b, H, H, relu=True, pool=POOL).wait()
y = j(x)
torch.cuda.synchronize()
y = j(x, out=y)
torch.cuda.synchronize()
print(j.info())
