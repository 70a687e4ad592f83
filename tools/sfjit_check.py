"""sfjit vs sf3x3 on the GPU: bit-identity on small random layers (relu/pool, ragged
batches whose CTA tile ranges cross images) and timing on VGG16 layer shapes.

python tools/sfjit_check.py [--time]
"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2212_08815_b200 import device, workloads as wl  # noqa: E402


def run_pair(c, k, h, n, relu, pool, zf=0.9, seed=0, flags=0):
    rng = np.random.default_rng(seed)
    w = (rng.standard_normal((k, c, 3, 3)) * 0.1).astype(np.float32)
    w[rng.random(w.shape) < zf] = 0
    b = (rng.standard_normal(k) * 0.1).astype(np.float32)
    x = rng.standard_normal((n, c, h, h)).astype(np.float32)
    xd = device.to_halo(torch.from_numpy(x).cuda())
    wd = torch.from_numpy(w).cuda()
    bank = device.sf_pack(wd)
    bt = torch.from_numpy(b).cuda()
    ref = device.sf_conv3x3(xd, bank, bt, relu=relu, pool=pool, w=h)
    t0 = time.time()
    j = device.SfJit(w, b, h, h, relu=relu, pool=pool, flags=flags).wait()
    dt = time.time() - t0
    got = j(xd)
    torch.cuda.synchronize()
    same = torch.equal(ref.view(torch.int32), got.view(torch.int32))
    return same, dt, j.info(), (ref, got)


def main():
    cases = [(3, 8, 8, 1, True, False), (16, 32, 16, 2, True, True), (24, 40, 12, 3, False, False),
             (64, 64, 28, 5, True, True), (32, 64, 14, 33, True, False), (8, 32, 56, 2, True, True),
             (64, 32, 224, 1, True, False)]
    cases = [cs + (0.9, 0, 0) for cs in cases] + [
        (64, 64, 56, 1, False, False, 0.95, 0, 8 | (1 << 16)), (24, 40, 12, 3, True, True, 0.9, 0, 4 | (1 << 16)),
        (16, 72, 28, 2, True, False, 0.8, 0, 16 | (8 << 8) | (1 << 16)),
        (32, 64, 14, 5, True, True, 0.9, 0, 0), (16, 48, 6, 7, True, True, 0.9, 0, 0), (3, 64, 30, 3, True, True, 0.5, 0, 0)]
    ok = True
    for cs in cases:
        same, dt, info, (ref, got) = run_pair(*cs)
        ok &= same
        d = (ref - got).abs().max().item()
        print(f"c={cs[0]} k={cs[1]} h={cs[2]} n={cs[3]} relu={cs[4]} pool={cs[5]}: bitwise={same} maxdiff={d:.3e} "
              f"compile {dt:.1f}s regs {info['registers']} cc {info['channels_per_chunk']} S {info['stages']} "
              f"bh {info['box_rows']} P {info['row_pitch']} nb {info['boxes_per_cta']}", flush=True)
    if "--time" in sys.argv:
        layers = wl.vgg16_weights(seed=103, zero_frac=0.9)
        shapes = wl.vgg16_conv_shapes()
        pools = [False, True, False, True, False, False, True, False, False, True, False, False, True]
        n = 32
        for li in [int(a) for a in sys.argv[sys.argv.index("--time") + 1].split(",")] if len(sys.argv) > sys.argv.index("--time") + 1 else [8]:
            (wt, b) = layers[li]
            k, c = wt.shape[:2]
            h = shapes[li][2] if isinstance(shapes[li], tuple) else None
            h = [224, 224, 112, 112, 56, 56, 56, 28, 28, 28, 14, 14, 14][li]
            x = torch.randn(n, c, h, h, device="cuda")
            xd = device.to_halo(x)
            wd = torch.from_numpy(wt).cuda()
            bank = device.sf_pack(wd)
            bt = torch.from_numpy(b).cuda()
            t0 = time.time()
            j = device.SfJit(wt, b, h, h, relu=True, pool=pools[li]).wait()
            ct = time.time() - t0
            out1 = device.sf_conv3x3(xd, bank, bt, relu=True, pool=pools[li], w=h)
            out2 = j(xd)
            torch.cuda.synchronize()
            same = torch.equal(out1.view(torch.int32), out2.view(torch.int32))
            nnz = int((wt != 0).sum())
            flops = 2 * nnz * n * h * h  # approx (ignores border taps)

            def tm(fn, reps=10):
                fn()
                torch.cuda.synchronize()
                a, bb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                for _ in range(reps):
                    fn()
                bb.record()
                bb.synchronize()
                return a.elapsed_time(bb) / reps

            t1 = tm(lambda: device.sf_conv3x3(xd, bank, bt, relu=True, pool=pools[li], out=out1, w=h))
            t2 = tm(lambda: j(xd, out=out2))
            print(f"L{li} {c}->{k} @{h} n={n}: bitwise={same} compile {ct:.1f}s  sf3x3 {t1*1e3:.0f} us "
                  f"({flops/t1/1e9:.1f} TF/s)  sfjit {t2*1e3:.0f} us ({flops/t2/1e9:.1f} TF/s)  info {j.info()}",
                  flush=True)
    print("ALL BITWISE OK" if ok else "MISMATCH")


if __name__ == "__main__":
    main()
