"""Shared-memory bank model of the sfjit patch loads: for each VGG16 row width, the
plan's tile-row padding, column block BW and row pitch P (mirroring make_plan), and the
wavefronts per warp-wide load (e0/e1: the 8-byte even pairs, o1/o2: the 4-byte odd
loads), averaged over the warps of an image.  2.0 is conflict-free for a 256-byte
(8-byte) load; the 28x28 rows without padding (14 tiles, BW = 2) give 2.85.

usage: python tools/sfjit_banks.py
"""
import itertools
def align(v,a): return (v+a-1)//a*a
def plan(w, padmode=1, BWo=None, Po=None):
    tprr = w//2
    tpr = align(tprr,8) if tprr%2 else tprr
    if padmode and 8 < tprr < 16: tpr = 16
    bw = 16
    while tpr % bw: bw >>= 1
    if BWo: bw = BWo
    P = align(2*tpr+2, 4)
    if bw < 16:
        while P % 32 != 16: P += 4
    if Po: P = Po
    return tpr, bw, P
def wavefronts(addrs, width):
    # addrs: float index per lane; width 1 or 2 floats
    banks = {}
    for a in addrs:
        for k in range(width):
            banks.setdefault((a+k) % 32, set()).add(a+k)
    need = max(len(v) for v in banks.values())
    return max(need, (len(addrs)*width*4 + 127)//128)
def layer(w, h, **kw):
    tpr, bw, P = plan(w, **kw)
    U = 2*tpr
    tot = {}
    nwarps = 0
    TPI = tpr*h
    for w0 in range(0, min(TPI, 32*64), 32):
        tts = range(w0, w0+32)
        rows, cols = [], []
        for tt in tts:
            r2, qq = divmod(tt, U)
            col = (qq // (2*bw))*bw + qq % bw
            par = (qq // bw) & 1
            rows.append(2*r2+par); cols.append(col)
        base = [r*P + 2*c for r, c in zip(rows, cols)]
        for name, off, wd in (("e0",0,2),("e1",2,2),("o1",1,1),("o2",2,1)):
            tot[name] = tot.get(name,0) + wavefronts([b+off for b in base], wd)
        nwarps += 1
    return tpr, bw, P, {k: round(v/nwarps,2) for k,v in tot.items()}
for w in (224,112,56,28,14):
    print(w, layer(w, w), layer(w,w,padmode=0))
