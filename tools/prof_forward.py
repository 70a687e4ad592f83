"""One VGG16 forward (config 3, batch 32) for ncu: two warm eager forwards, then one
inside an NVTX range 'profiled' (ncu --nvtx --nvtx-include 'profiled/').  Eager (no CUDA
graph), one batch part, so every kernel launch is one full-batch layer group.

  ncu --nvtx --nvtx-include "profiled/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
      dram__bytes_write.sum --clock-control none --csv python tools/prof_forward.py
"""
import os
import sys

os.environ["FSCNN_GRAPHS"] = "0"
os.environ["FSCNN_PARTS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_08815_b200 import workloads as wl  # noqa: E402
from paper_2212_08815_b200.engine import VGGEngine  # noqa: E402

eng = VGGEngine(wl.vgg16_weights(seed=103, zero_frac=0.9), batch=32, hw=224).wait_compiled()
x = torch.from_numpy(wl.vgg16_input(32, seed=104)).cuda()
for _ in range(2):
    eng.forward_device(x)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
eng.forward_device(x)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("groups per layer:", [st.jit.info()["groups"] if st.jit else 0 for st in eng.steps])
