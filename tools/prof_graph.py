"""One VGG16 step (config 3, batch 32) exactly as bench.py times it -- the engine's CUDA
graph: L0/L1 full batch, 8 batch parts on concurrent streams from L2 on -- for ncu's
whole-graph mode.  Three warm replays, then one inside an NVTX range 'profiled'.

  ncu --graph-profiling graph --nvtx --nvtx-include "profiled/" --cache-control none \\
      --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
      dram__bytes_write.sum,lts__t_bytes.sum --csv python tools/prof_graph.py

The graph is profiled as ONE workload (its kernels keep their concurrency and share the
L2 as in the bench; caches are not flushed), so dram__bytes is the step's real DRAM
traffic -- against the serialised, cold-cache launch list of tools/prof_forward.py, where
every group kernel of a layer re-reads the layer's input from DRAM.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_08815_b200 import workloads as wl  # noqa: E402
from paper_2212_08815_b200.engine import VGGEngine  # noqa: E402

n = int(os.environ.get("N", "32"))
eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=n, hw=224).wait_compiled()
x = torch.from_numpy(wl.vgg16_input(n, seed=104)).cuda()
xh = eng.stage_input(x)
for _ in range(4):
    eng.run(xh)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
eng.run(xh)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    eng.run(xh)
b.record()
b.synchronize()
print("parts", eng.parts_for(n), "ms/step (not a bench value under ncu)", a.elapsed_time(b) / 5)
