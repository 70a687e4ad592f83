"""Where the public-API (e2e) forward of the VGG16 stack spends its time.

Times network.forward(prepared, list[DenseTensor3]) for batch 32 and each piece of
it separately (host packing into pinned memory, H2D, layout conversion, the stack,
output conversion, D2H, host unpacking), with a device sync around each piece.

usage: python tools/e2e_profile.py [BATCH] [REPS]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2212_08815_b200 import device, network, workloads as wl
from paper_2212_08815_b200.engine import VGGEngine
from paper_2212_08815_b200.sparse_core import DenseTensor3

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=n, hw=224)
prepared = network.prepared_from_engine(eng)
x_np = wl.vgg16_input(n, seed=104)
batch = [DenseTensor3.from_array(x_np[i]) for i in range(n)]
for _ in range(3):
    network.forward(prepared, batch)
torch.cuda.synchronize()


def timed(fn, reps=reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3


c, h, w = 3, 224, 224
h_in = torch.empty(n * c * h * w, dtype=torch.float32).pin_memory()
np_in = h_in.numpy().reshape(n, -1)
d_in = torch.empty(n * c * h * w, dtype=torch.float32, device="cuda")
oc, ohw = eng.out_c, eng.out_hw
h_out = torch.empty(n * oc * ohw * ohw, dtype=torch.float32).pin_memory()


def pack():
    for i, t in enumerate(batch):
        np_in[i] = t.data


pinned = network.pinned_batch(n, (3, 224, 224))
for i in range(n):
    pinned[i].data[:] = batch[i].data
d_w = torch.empty(n * 3 * 224 * 224, dtype=torch.float32, device="cuda")
res = {
    "forward_total_pinned": timed(lambda: network.forward(prepared, pinned)),
    "forward_whc": timed(lambda: eng.forward_whc(d_w, n)),
    "forward_total": timed(lambda: network.forward(prepared, batch)),
    "host_pack": timed(pack),
    "h2d": timed(lambda: d_in.copy_(h_in, non_blocking=True)),
    "whc_to_nchw": timed(lambda: device.whc_to_nchw(d_in, n, c, h, w)),
}
x = device.whc_to_nchw(d_in, n, c, h, w)
res["stage_input"] = timed(lambda: eng.stage_input(x))
xh = eng.stage_input(x)
res["stack"] = timed(lambda: eng.run(xh))
y = eng.forward_device(x)
res["nchw_to_whc"] = timed(lambda: device.nchw_to_whc(y.contiguous()))
whc = device.nchw_to_whc(y.contiguous())
res["d2h"] = timed(lambda: h_out.copy_(whc.view(-1), non_blocking=True))
out = h_out.numpy().reshape(n, -1)
res["host_unpack"] = timed(lambda: [DenseTensor3((oc, ohw, ohw), out[i].copy()) for i in range(n)])
res["check_batch"] = timed(lambda: network._check_batch(prepared, batch))
print({k: round(v, 3) for k, v in res.items()})
print("img/s e2e", n / res["forward_total"] * 1e3, " sum of parts", round(sum(v for k, v in res.items() if k != "forward_total"), 3))
