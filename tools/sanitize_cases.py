"""Smallest cases that exercise every hand-written kernel once, for compute-sanitizer
(memcheck / racecheck / synccheck).  Run it bare first; then under one tool at a time:

  compute-sanitizer --tool racecheck --racecheck-report hazard python tools/sanitize_cases.py

Kernels: the encoder (count / scan / write) and decoder, sf_exact, sf3x3 (KT 1/2/4,
fused ReLU+pool), the specialised sfjit kernels (part and multi-image CTA modes, pool),
the sparse-input strip / smem / gather / channel-major kernels, ReLU, pool, layouts.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FSCNN_GRAPHS", "0")
from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402
from paper_2212_08815_b200.engine import VGGEngine  # noqa: E402

torch.cuda.set_device(0)
rng = np.random.default_rng(0)


def t(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# encoder / decoder (all orders on one tensor)
x = rng.standard_normal((2, 5, 9, 11)).astype(np.float32)
x[rng.random(x.shape) < 0.7] = 0
for order in ("CHW", "WHC", "HWC"):
    enc = device.encode_order(t(x), order)
    back = device.decode_order(enc.nodes, enc.seg_off, x.shape, order)
assert torch.equal(back.cpu(), torch.from_numpy(np.where(x == 0, 0, x).astype(np.float32)))

# sparse-filter: exact kernel, jump-table kernel at KT 1/2/4 with ReLU+pool, sfjit
c, k, h = 12, 40, 16
w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
w[rng.random(w.shape) < 0.85] = 0
b = (rng.standard_normal(k) * 0.1).astype(np.float32)
xs = rng.standard_normal((3, c, h, h)).astype(np.float32)
enc = device.encode_order(t(w), "CHW")
device.sf_conv_exact(t(xs), enc.nodes, enc.seg_off, k, 3, 3, 1, 1, t(b))
xh = device.to_halo(t(xs))
outs = []
for kt in (1, 2, 4):
    outs.append(device.sf_conv3x3(xh, device.sf_pack(t(w), kt), t(b), relu=True, pool=True, w=h).cpu())
jit = device.SfJit(w, b, h, h, relu=True, pool=True)
outs.append(jit(xh).cpu())
jit2 = device.SfJit(w, b, 6, 6, relu=True, pool=False)  # multi-image CTAs, ragged last CTA
jit2(device.to_halo(t(rng.standard_normal((5, c, 6, 6)).astype(np.float32))))
assert all(torch.equal(o, outs[0]) for o in outs)

# sparse-input kernels: strip (L2 and smem banks), gather (stride 2), channel-major
xi, wi, _ = wl.c2()
xi, wi = xi[:, :32, :12, :12].copy(), wi[:64, :32].copy()
enc = device.encode_order(t(xi), "CHW")
n_, ci, hi, wd = xi.shape
device.si_conv3x3(enc.nodes, enc.seg_off, n_, ci, hi, wd, device.si_pack3x3(t(wi)), 64)
device.si_conv3x3_fast(enc.nodes, enc.seg_off, n_, ci, hi, wd, device.si_pack_fast(t(wi)), 64)
device.si_conv(enc.nodes, enc.seg_off, n_, ci, hi, wd, device.kcrs_to_crsk(t(wi)), 64, 3, 3, 2, 1)

# the fused VGG stack (sfjit + jump-table fallback for odd sizes) and elementwise ops
layers = wl.vgg16_weights(seed=1, zero_frac=0.9, scale=0.0625)
eng = VGGEngine(layers, batch=2, hw=32)
y = eng.forward_device(t(wl.vgg16_input(2, seed=2, hw=32)))
device.relu(t(xs))
device.pool2d(t(xs), 2, 2, True)
torch.cuda.synchronize()
print("sanitize cases ok", tuple(y.shape))
