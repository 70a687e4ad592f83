"""Time sfjit plan variants on VGG16 layer shapes (batch 32, 90 % filter zeros by default).

usage: python tools/sfjit_variants.py LAYERS VARIANT [VARIANT ...]
  LAYERS   comma list, e.g. 1,5,8,11
  VARIANT  NAME:KEY=VAL,KEY=VAL  (keys are FSCNN_SFJIT_* suffixes: KT, WMAX, SMEM_KB, MINB, ...)
           e.g. base:  w8:WMAX=8,SMEM_KB=105,MINB=2
Env: ZF (zero fraction, 0.9), N (batch, 32), REPS (7).
Prints one line per (layer, variant): ms, nnz-TF/s, fraction of the 72.3 TF/s FFMA peak, plan.
Each variant is checked bit for bit against the first variant's output.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402

PEAK = 72.3
zf = float(os.environ.get("ZF", "0.9"))
n = int(os.environ.get("N", "32"))
reps = int(os.environ.get("REPS", "7"))
layers = [int(v) for v in sys.argv[1].split(",")]
variants = []
for spec in sys.argv[2:]:
    name, _, kv = spec.partition(":")
    env = dict(item.split("=", 1) for item in kv.split(",") if item)
    variants.append((name, env))
KEYS = ("KT", "WMAX", "SMEM_KB", "MINB", "ODD", "NOBAR", "TMA_HINT", "STORE_CS", "REPEAT", "PADTPR", "TMA_SPLIT", "REALP", "TMA_MERGE", "UNI")


def time_fn(fn):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


for li in layers:
    c, k, h, w = wl.vgg16_conv_shapes()[li]
    x, wt, b = wl.sweep_layer(li, "sf", zf, n=n)
    xh = device.to_halo(torch.from_numpy(x).cuda())
    pool = li in (1, 3, 6, 9, 12)
    nz = (wt != 0)
    # in-bounds multiplies: per tap, the rows/cols of the output that see an in-bounds input
    inb = np.array([[(h - abs(kh - 1)) * (w - abs(kw - 1)) for kw in range(3)] for kh in range(3)], np.float64)
    fl = 2.0 * n * float((nz.sum(axis=(0, 1)) * inb).sum())
    ref = None
    for name, env in variants:
        for key in KEYS:
            os.environ.pop("FSCNN_SFJIT_" + key, None)
        for key, val in env.items():
            os.environ["FSCNN_SFJIT_" + key] = val
        try:
            jit = device.SfJit(wt, b, h, w, relu=True, pool=pool).wait()
        except Exception as e:  # noqa: BLE001
            print(f"L{li:2d} {name:10s} plan failed: {e}", flush=True)
            continue
        out = jit(xh)
        ms = time_fn(lambda: jit(xh, out=out))
        torch.cuda.synchronize()
        same = ""
        if ref is None:
            ref = out.clone()
        else:
            same = "bitwise" if torch.equal(out.view(torch.int32), ref.view(torch.int32)) else "DIFF"
        tf = fl / (ms * 1e-3) / 1e12
        inf = jit.info()
        print(f"L{li:2d} {c:3d}->{k:3d}@{h:3d} {name:10s} {ms:7.4f} ms {tf:6.2f} TF/s {tf / PEAK:5.3f}  "
              f"warps {inf['warps']} kt {inf['filters_per_group']} cc {inf['channels_per_chunk']} S {inf['stages']} "
              f"smem {inf['smem_bytes'] // 1024}K regs {inf['registers']} mode {inf['ctas_per_image_or_minus_images_per_cta']} {same}",
              flush=True)
        del jit, out
    del xh, ref
    torch.cuda.empty_cache()
