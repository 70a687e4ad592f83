"""Prototype v3: straight-line sparse-filter code, FFMA2 with immediate weights.
Lane = 2x2 output tile (acc pairs = the two columns of a row), warp = KT filters.
Patch = 4 rows x 4 cols as b64 pairs (c0,c1),(c2,c3) + odd pair (c1,c2) built by mov.
python gen3.py C W G DENS SPLIT NT MINB KT > k.ptx
"""
import random, struct, sys
C, W, G, DENS, SPLIT, NT, MINB, KT = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]),
    int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8]))
ODD = int(sys.argv[9]) if len(sys.argv) > 9 else 1
P = W + 8
TPR = W // 2
ROWS = 24
CH_FLOATS = ROWS * P
random.seed(7)
out = []; e = out.append
e(".version 8.7\n.target sm_100a\n.address_size 64\n")
e(".extern .shared .align 16 .b8 smem[];")
nff = 0
for g in range(G):
    e(f".visible .entry k{g}(.param .u64 py, .param .u32 ptiles) .maxntid {NT} .minnctapersm {MINB} {{")
    e(f".reg .b64 a<{KT*2}>; .reg .b64 e<8>; .reg .b64 o<4>; .reg .f32 h<16>; .reg .b64 ry, rt, dw; .reg .f32 fw; .reg .b32 rs, rl, rb, rt0, rty, rtx, rq; .reg .pred q;")
    e("ld.param.u64 ry, [py];")
    e("mov.u32 rs, smem;")
    e("mov.u32 rl, %tid.x; mov.u32 rb, %ctaid.x;")
    e("and.b32 rt0, rl, 127;")
    e(f"mul.lo.u32 rty, rt0, {(1<<16)//TPR + 1}; shr.u32 rty, rty, 16; mul.lo.u32 rtx, rty, {TPR}; sub.u32 rtx, rt0, rtx;")
    e(f"mul.lo.u32 rq, rty, {2*P*4}; mad.lo.u32 rq, rtx, 8, rq; add.u32 rs, rs, rq;")
    e("setp.eq.u32 q, rb, 0x7fffffff;")
    for i in range(KT * 2):
        e(f"mov.b64 a{i}, 0;")
    for c in range(C):
        if SPLIT and c and c % SPLIT == 0:
            e("@q bra.uni END;")
        cb = (c % 16) * CH_FLOATS * 4
        for r in range(4):
            e(f"ld.shared.b64 e{r*2}, [rs+{cb + r*P*4}];")
            e(f"ld.shared.b64 e{r*2+1}, [rs+{cb + r*P*4 + 8}];")
        nz = []
        for kl in range(KT):
            for t in range(9):
                if random.random() < DENS:
                    nz.append((kl, t, struct.unpack("<I", struct.pack("<f", random.gauss(0, 0.05)))[0]))
        need_odd = {t // 3 + py for (kl, t, w) in nz if t % 3 == 1 for py in range(2)}
        for r in (sorted(need_odd) if ODD else []):
            e(f"{{ .reg .f32 x0, x1, x2, x3; mov.b64 {{x0, x1}}, e{r*2}; mov.b64 {{x2, x3}}, e{r*2+1}; mov.b64 o{r}, {{x1, x2}}; }}")
        for kl, t, hx in nz:
            kh, kw = divmod(t, 3)
            nff += 4
            e(f"mov.b32 fw, 0f{hx:08X}; mov.b64 dw, {{fw, fw}};")
            for py in range(2):
                a = f"a{kl*2+py}"
                r = py + kh
                if kw != 1 or ODD:
                    src = f"e{r*2 + kw//2}" if kw != 1 else f"o{r}"
                    e(f"fma.rn.f32x2 {a}, {src}, dw, {a};")
                else:
                    e(f"{{ .reg .f32 x0, x1, x2, x3, s0, s1; mov.b64 {{x0, x1}}, e{r*2}; mov.b64 {{x2, x3}}, e{r*2+1}; mov.b64 {{s0, s1}}, {a};")
                    e(f"fma.rn.f32 s0, x1, fw, s0; fma.rn.f32 s1, x2, fw, s1; mov.b64 {a}, {{s0, s1}}; }}")
    e("END:")
    e("mad.wide.u32 rt, rb, 8192, ry; mul.wide.u32 ry, rl, 8; add.u64 rt, rt, ry;")
    for i in range(1, KT * 2):
        e(f"add.rn.f32x2 a0, a0, a{i};")
    e("st.global.b64 [rt], a0;")
    e("ret;}")
print("\n".join(out))
print(f"// ffma_per_group {nff // G}", file=sys.stderr)
