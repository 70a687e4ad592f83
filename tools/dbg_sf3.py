"""Debug harness: run the fast sparse-filter kernel on config 1 in a given debug mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2212_08815_b200 import device, workloads as wl

x, w, b = wl.c1()
xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
enc = device.encode_order(wt, "CHW")
ref = device.sf_conv_exact(xt, enc.nodes, enc.seg_off, 64, 3, 3, 1, 1, None)
bank = device.sf_pack(wt)
print("bank total", bank.total, "nnz", bank.nnz, "plan", bank.chunk_plan(device.pick_ly(bank.c, 56)), flush=True)
for ly in (2, 4, 8):
    y = device.from_halo(device.sf_conv3x3(device.to_halo(xt), bank, None, relu=False, pool=False, w=56, ly=ly), 56)
    torch.cuda.synchronize()
    err = float((y - ref).abs().max() / ref.abs().max())
    print(f"mode {os.environ.get('FSCNN_SF3_DEBUG','0')} ly {ly}: normwise err {err:.3e}", flush=True)
