"""Time the VGG16 stack (batch 32, 90 %) with the batch on 1, 2 or 4 streams."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2212_08815_b200 import workloads as wl
from paper_2212_08815_b200.engine import VGGEngine

eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=32, hw=224)
x = torch.from_numpy(wl.vgg16_input(32, seed=104)).cuda()
xh = eng.stage_input(x)
ref = eng.run(xh).clone()
for parts in (1, 2, 4, 1, 2):
    fn = lambda: eng.run(xh, parts)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        y = fn()
    b.record(); b.synchronize()
    same = torch.equal(y, ref)
    print(f"parts {parts}: {a.elapsed_time(b) / 10:.3f} ms  identical={same}", flush=True)

# the same stack captured once in a CUDA graph (both streams), then replayed
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    eng.run(xh, 2)
torch.cuda.current_stream().wait_stream(s)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    yg = eng.run(xh, 2)
for _ in range(3):
    g.replay()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    g.replay()
b.record(); b.synchronize()
print(f"graph, parts 2: {a.elapsed_time(b) / 10:.3f} ms  identical={torch.equal(yg, ref)}", flush=True)
