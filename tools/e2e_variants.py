"""e2e forward (pinned inputs) timed the way bench.py does it, a few variants."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_08815_b200 import network, workloads as wl
from paper_2212_08815_b200.engine import VGGEngine
from paper_2212_08815_b200.sparse_core import DenseTensor3

eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=32, hw=224)
prepared = network.prepared_from_engine(eng)
x_np = wl.vgg16_input(32, seed=104)
batch = network.pinned_batch(32, (3, 224, 224))
for i in range(32):
    batch[i].data[:] = DenseTensor3.from_array(x_np[i]).data
for _ in range(3):
    network.forward(prepared, batch)
torch.cuda.synchronize()
for label in ("keep result", "drop result", "keep result"):
    t0 = time.perf_counter()
    res = None
    for _ in range(10):
        r = network.forward(prepared, batch)
        if label == "keep result":
            res = r
    dt = (time.perf_counter() - t0) / 10
    print(f"{label:12s}: {dt * 1e3:.3f} ms/step  {32 / dt:.0f} img/s", flush=True)
