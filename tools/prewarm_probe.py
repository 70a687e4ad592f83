"""Time the sfjit dry pass (prewarm) of one VGG16 layer alone and next to the previous layer."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402

ws = wl.vgg16_weights(seed=103, zero_frac=0.9)
H = [224, 224, 112, 112, 56, 56, 56, 28, 28, 28, 14, 14, 14]
P = [False, True, False, True, False, False, True, False, False, True, False, False, True]
li = int(sys.argv[1]) if len(sys.argv) > 1 else 8
jits = {i: device.SfJit(ws[i][0], ws[i][1], H[i], H[i], relu=True, pool=P[i]).wait() for i in (li - 1, li)}
s = torch.cuda.Stream()
for _ in range(2):
    with torch.cuda.stream(s):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        jits[li].prewarm(s)
        b.record()
    b.synchronize()
    print(f"prewarm L{li} alone: {a.elapsed_time(b):.3f} ms", flush=True)
n = 32
x = device.to_halo(torch.randn(n, ws[li - 1][0].shape[1], H[li - 1], H[li - 1], device="cuda"))
y = jits[li - 1](x)
torch.cuda.synchronize()
for warm in (False, True):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    if warm:
        jits[li].prewarm(s)
    jits[li - 1](x, out=y)
    b.record()
    b.synchronize()
    torch.cuda.synchronize()
    print(f"L{li-1} with prewarm of L{li}={warm}: {a.elapsed_time(b):.3f} ms", flush=True)
