"""Seeded random-shape fuzz of the fast kernels against the bit-exact ones (which the
tests pin to the reference): the sparse-filter kernel (every filters-per-warp / CTA
plan, with and without the fused ReLU + pool) against the reference-order kernel, the
specialised per-layer kernels (sfjit: per-group and fused modes) bit for bit against the
jump-table kernel, and the channel-major sparse-input kernel against the strip kernel.  Reports the worst
normwise error (north-star bar 1e-4) and any plan disagreement (must be bit-identical).

usage: python tools/fuzz_parity.py [--cases 200] [--seed 1]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2212_08815_b200 import device


def nerr(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", type=int, default=200)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--sfjit-every", type=int, default=1, help="check the specialised kernels every Nth case (0: off)")
    args = ap.parse_args()
    rng = np.random.default_rng(args.seed)
    worst_sf = worst_si = 0.0
    plan_mismatch = 0
    sfjit_cases = sfjit_mismatch = 0
    for i in range(args.cases):
        n = int(rng.integers(1, 5))
        c = int(rng.choice([1, 3, 5, 16, 17, 33, 64, 100]))
        k = int(rng.choice([1, 3, 8, 31, 32, 33, 64, 70, 128, 130]))
        h = int(rng.integers(1, 40)) * (2 if rng.random() < 0.5 else 1)
        w = int(rng.integers(1, 40)) * (2 if rng.random() < 0.5 else 1)
        zf = float(rng.choice([0.0, 0.5, 0.9, 0.97, 1.0]))
        x = rng.standard_normal((n, c, h, w)).astype(np.float32)
        wt = rng.standard_normal((k, c, 3, 3)).astype(np.float32)
        wt[rng.random(wt.shape) < zf] = 0
        bias = rng.standard_normal(k).astype(np.float32)
        xd, wd, bd = (torch.from_numpy(a).cuda() for a in (x, wt, bias))
        # sparse filter: exact reference-order kernel vs every plan of the fast kernel
        enc = device.encode_order(wd, "CHW")
        ref = device.sf_conv_exact(xd, enc.nodes, enc.seg_off, k, 3, 3, 1, 1, bd, relu=True)
        xh = device.to_halo(xd)
        pool = h % 2 == 0 and w % 2 == 0 and rng.random() < 0.5
        outs = []
        for kt, warps in ((4, 0), (2, 0), (2, 4), (1, 0), (8, 0)):
            bank = device.sf_pack(wd, kt)
            y = device.sf_conv3x3(xh, bank, bd, relu=True, pool=False, w=w, cta_warps=warps)
            got = device.from_halo(y, w)
            worst_sf = max(worst_sf, nerr(got, ref))
            if pool:
                yp = device.sf_conv3x3(xh, bank, bd, relu=True, pool=True, w=w, cta_warps=warps)
                outs.append(device.from_halo(yp, w // 2).clone())
            outs.append(got.clone())
        # the specialised kernels (per-group launches at 48 / 16 filters per group, and the
        # fused one-kernel mode the layer API uses) on even extents: bit-identical to the
        # jump-table kernel (same per-output order), pooled and not
        if h % 2 == 0 and w % 2 == 0 and (args.sfjit_every and i % args.sfjit_every == 0):
            base = outs[0] if not pool else outs[1]
            for flags in (0, 16, 4 | (8 << 8) | (1 << 16)):
                jit = device.SfJit(wd, bd, h, w, relu=True, pool=False, flags=flags).wait()
                yj = device.from_halo(jit(xh), w)
                sfjit_cases += 1
                if not torch.equal(yj.contiguous().view(torch.int32), base.contiguous().view(torch.int32)):
                    sfjit_mismatch += 1
                if pool:
                    jp = device.SfJit(wd, bd, h, w, relu=True, pool=True, flags=flags).wait()
                    yp = device.from_halo(jp(xh), w // 2)
                    if not torch.equal(yp.contiguous().view(torch.int32), outs[0].contiguous().view(torch.int32)):
                        sfjit_mismatch += 1
        # all plans bit-identical
        per_plan = len(outs) // 5
        for j in range(1, 5):
            for q in range(per_plan):
                if not torch.equal(outs[q].view(torch.int32), outs[j * per_plan + q].view(torch.int32)):
                    plan_mismatch += 1
        # sparse input: channel-major vs strip kernel
        xs = np.abs(x)
        xs[rng.random(xs.shape) < float(rng.choice([0.0, 0.5, 0.9, 1.0]))] = 0
        xsd = torch.from_numpy(xs).cuda()
        enc_i = device.encode_order(xsd, "CHW")
        wdense = torch.from_numpy(rng.standard_normal((k, c, 3, 3)).astype(np.float32)).cuda()
        a = device.si_conv3x3(enc_i.nodes, enc_i.seg_off, n, c, h, w, device.si_pack3x3(wdense), k, bd)
        b = device.si_conv3x3_fast(enc_i.nodes, enc_i.seg_off, n, c, h, w, device.si_pack_fast(wdense), k, bd)
        worst_si = max(worst_si, nerr(b, a))
    torch.cuda.synchronize()
    print(f"{args.cases} cases: worst normwise SF fast vs exact {worst_sf:.2e}, SI channel-major vs strip "
          f"{worst_si:.2e}, plan mismatches {plan_mismatch}, specialised-kernel launches {sfjit_cases} "
          f"with {sfjit_mismatch} mismatches vs the jump-table kernel")
    assert worst_sf <= 1e-4 and worst_si <= 1e-4 and plan_mismatch == 0 and sfjit_mismatch == 0


if __name__ == "__main__":
    main()
