"""Per-layer times of the VGG16 stack (batch 32, 90 %): in-stack vs hot-repeat vs graph.

python tools/stack_probe.py
"""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2212_08815_b200 import workloads as wl  # noqa: E402
from paper_2212_08815_b200.engine import VGGEngine  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=n, hw=224).wait_compiled()
x = torch.from_numpy(wl.vgg16_input(n, seed=104)).cuda()
for _ in range(3):
    eng.forward_device(x)
torch.cuda.synchronize()


def ev():
    return torch.cuda.Event(enable_timing=True)


a, b = ev(), ev()
a.record()
for _ in range(10):
    eng.forward_device(x)
b.record()
b.synchronize()
print(f"stack: {a.elapsed_time(b) / 10:.3f} ms/step")

bufs = eng._buffers(n)
xh = eng.stage_input(x)


def layer_times(reps_inner):
    out = []
    cur, w = xh, 224
    for st, o in zip(eng.steps, bufs):
        st.conv(cur, o, w, n)
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record()
        for _ in range(reps_inner):
            st.conv(cur, o, w, n)
        b.record()
        b.synchronize()
        out.append(a.elapsed_time(b) / reps_inner)
        cur, w = o, (w // 2 if st.pool else w)
    return out


print("in-stack once :", [round(v, 3) for v in layer_times(1)])
print("hot x10       :", [round(v, 3) for v in layer_times(10)])

# (forward_device already replays a CUDA graph per batch size: engine.VGGEngine._run)
