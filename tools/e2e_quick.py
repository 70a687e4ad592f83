"""network.forward (pinned host inputs) ms per batch, and the device-only forward."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_08815_b200 import network, workloads as wl  # noqa: E402
from paper_2212_08815_b200.engine import VGGEngine  # noqa: E402
from paper_2212_08815_b200.sparse_core import DenseTensor3  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=n, hw=224).wait_compiled()
prepared = network.prepared_from_engine(eng)
x_np = wl.vgg16_input(n, seed=104)
batch = network.pinned_batch(n, (3, 224, 224))
for i in range(n):
    batch[i].data[:] = DenseTensor3.from_array(x_np[i]).data
for _ in range(3):
    network.forward(prepared, batch)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    network.forward(prepared, batch)
e2e = (time.perf_counter() - t0) / 10 * 1e3
x = torch.from_numpy(x_np).cuda()
for _ in range(3):
    eng.forward_device(x)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    eng.forward_device(x)
b.record()
b.synchronize()
t1 = time.perf_counter()
for _ in range(10):
    eng.forward_device(x)
    torch.cuda.synchronize()
sync_dev = (time.perf_counter() - t1) / 10 * 1e3
print(f"n={n} e2e {e2e:.3f} ms ({n / e2e * 1e3:.0f} img/s)  device {a.elapsed_time(b) / 10:.3f} ms  "
      f"device+sync per call {sync_dev:.3f} ms")
