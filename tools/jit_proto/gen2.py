"""Prototype v2: straight-line sparse-filter code, weights as immediates.
Lane = 2x2 output tile, warp = KT filters x 32 tiles.  MODE 'ffma': 4 scalar FFMA-imm per
nonzero; 'ffma2': kw in {0,2} -> mov imm + 2 FFMA2 (broadcast weight), kw = 1 -> 4 FFMA.
python gen2.py C W G DENS SPLIT NT MINB KT MODE
"""
import random, struct, sys
C, W, G, DENS, SPLIT, NT, MINB, KT, MODE = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4]),
    int(sys.argv[5]), int(sys.argv[6]), int(sys.argv[7]), int(sys.argv[8]), sys.argv[9])
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
    e(f".reg .b64 a<{KT*2}>; .reg .f32 p<16>; .reg .b64 pp<8>; .reg .b64 ry, rt, dw; .reg .f32 fw; .reg .b32 rs, rl, rb, rt0, rty, rtx, rq; .reg .pred q;")
    e("ld.param.u64 ry, [py];")
    e("mov.u32 rs, smem;")
    e("mov.u32 rl, %tid.x; mov.u32 rb, %ctaid.x;")
    e("rem.u32 rt0, rl, 128;")
    e(f"div.u32 rty, rt0, {TPR}; rem.u32 rtx, rt0, {TPR};")
    e(f"mul.lo.u32 rq, rty, {2*P*4}; mad.lo.u32 rq, rtx, 8, rq; add.u32 rs, rs, rq;")
    e("setp.eq.u32 q, rb, 0x7fffffff;")
    for i in range(KT * 2):
        e(f"mov.b64 a{i}, 0;")
    for c in range(C):
        if SPLIT and c and c % SPLIT == 0:
            e("@q bra.uni END;")
        cb = (c % 16) * CH_FLOATS * 4
        for r in range(4):
            e(f"ld.shared.v2.f32 {{p{r*4}, p{r*4+1}}}, [rs+{cb + r*P*4}];")
            e(f"ld.shared.v2.f32 {{p{r*4+2}, p{r*4+3}}}, [rs+{cb + r*P*4 + 8}];")
            e(f"mov.b64 pp{r*2}, {{p{r*4}, p{r*4+1}}}; mov.b64 pp{r*2+1}, {{p{r*4+2}, p{r*4+3}}};")
        for kl in range(KT):
            for t in range(9):
                if random.random() < DENS:
                    kh, kw = divmod(t, 3)
                    hx = struct.unpack("<I", struct.pack("<f", random.gauss(0, 0.05)))[0]
                    nff += 4
                    for py in range(2):
                        a = f"a{kl*2+py}"
                        r = py + kh
                        if MODE == "ffma2" and kw != 1:
                            e(f"mov.b32 fw, 0f{hx:08X}; mov.b64 dw, {{fw, fw}};")
                            e(f"fma.rn.f32x2 {a}, dw, pp{r*2 + kw//2}, {a};")
                        else:
                            e(f"{{ .reg .f32 x, y; mov.b64 {{x, y}}, {a};")
                            e(f"fma.rn.f32 x, p{r*4 + kw}, 0f{hx:08X}, x; fma.rn.f32 y, p{r*4 + kw + 1}, 0f{hx:08X}, y;")
                            e(f"mov.b64 {a}, {{x, y}}; }}")
    e("END:")
    e("mad.wide.u32 rt, rb, 4096, ry; mul.wide.u32 ry, rl, 8; add.u64 rt, rt, ry;")
    for i in range(1, KT * 2):
        e(f"add.rn.f32x2 a0, a0, a{i};")
    e("st.global.b64 [rt], a0;")
    e("ret;}")
print("\n".join(out))
print(f"// ffma_per_group {nff // G}", file=sys.stderr)
