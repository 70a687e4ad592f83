"""Prototype: straight-line sparse-filter code (weights as FFMA immediates) for one
VGG16 layer shape, one kernel per 32-filter group.  Lane = 2x2 output tile, warp = 32
filters x 32 tiles, CTA = 4 warps.  Input patches come from a static 16-channel smem
region (no TMA: measures the inner loop only).  Perf prototype -- no correctness.

python gen.py C W GROUPS DENSITY SPLIT > k.ptx
"""
import random
import struct
import sys

C, W, G, DENS, SPLIT = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]), int(sys.argv[5])
NT, MINB = int(sys.argv[6]), int(sys.argv[7])
KT = 32
P = W + 8  # row pitch (floats)
TPR = W // 2  # tiles per row
ROWS = 24
CH_FLOATS = ROWS * P
random.seed(7)
out = []
e = out.append
e(".version 8.7\n.target sm_100a\n.address_size 64\n")
e(".extern .shared .align 16 .b8 smem[];")
for g in range(G):
    e(f".visible .entry k{g}(.param .u64 py, .param .u32 ptiles) .maxntid {NT} .minnctapersm {MINB} {{")
    e(f".reg .f32 a<{KT*4}>; .reg .f32 p<16>; .reg .b64 ry, rt; .reg .b32 rs, rl, rw, rb, rt0, rty, rtx, rq; .reg .pred q;")
    e("ld.param.u64 ry, [py];")
    e("mov.u32 rs, smem;")
    e("mov.u32 rl, %tid.x; mov.u32 rb, %ctaid.x;")
    # tile index within the CTA's range (128 tiles) -> row/col relative to the CTA band
    e("rem.u32 rt0, rl, 128;")
    e(f"div.u32 rty, rt0, {TPR}; rem.u32 rtx, rt0, {TPR};")
    e(f"mul.lo.u32 rq, rty, {2*P*4}; mad.lo.u32 rq, rtx, 8, rq; add.u32 rs, rs, rq;")
    e("setp.eq.u32 q, rb, 0x7fffffff;")
    for i in range(KT * 4):
        e(f"mov.f32 a{i}, 0f00000000;")
    for c in range(C):
        if SPLIT and c and c % SPLIT == 0:
            e("@q bra.uni END;")
        cb = (c % 16) * CH_FLOATS * 4
        for r in range(4):
            e(f"ld.shared.v2.f32 {{p{r*4}, p{r*4+1}}}, [rs+{cb + r*P*4}];")
            e(f"ld.shared.v2.f32 {{p{r*4+2}, p{r*4+3}}}, [rs+{cb + r*P*4 + 8}];")
        for kl in range(KT):
            for t in range(9):
                if random.random() < DENS:
                    kh, kw = divmod(t, 3)
                    hx = struct.unpack("<I", struct.pack("<f", random.gauss(0, 0.05)))[0]
                    for py in range(2):
                        for px in range(2):
                            a = kl * 4 + py * 2 + px
                            e(f"fma.rn.f32 a{a}, p{(py+kh)*4 + px + kw}, 0f{hx:08X}, a{a};")
    e("END:")
    e("mad.wide.u32 rt, rb, 512, ry; mul.wide.u32 ry, rl, 4; add.u64 rt, rt, ry;")
    e("add.f32 a0, a0, a1;")
    for i in range(2, KT * 4):
        e(f"add.f32 a0, a0, a{i};")
    e("st.global.f32 [rt], a0;")
    e("ret;}")
print("\n".join(out))
