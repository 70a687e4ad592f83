"""Generates si3x3_cases.inc: the per-channel apply loop of si3x3_fast_kernel, as one
inline-PTX block with a real jump table.

For an output tile of TY x TX pixels the kernel reads the (TY+2) x (TX+2) input region
around it; the input at region position (ry, rx) feeds output (ry - kh, rx - kw) through
tap (kh, kw) for every tap that lands in the tile.  Which accumulators a position
touches is fixed, so each position gets its own block of FMAs with named registers,
reached by one `brx.idx` per nonzero input (a C++ switch compiles to a compare tree
with small jump tables at its leaves: ~6 extra branches per nonzero).

Arithmetic: scalar FMAs on 32-bit accumulators (64-bit pair accumulators with
fma.rn.f32x2 for the aligned column pairs were measured: ptxas then inserts ~4 register
moves per nonzero at the jump-table join, more than the pairs save).

Protocol (C++ wrapper si_chan<TY, TX>): the channel's entries {pos, value bits} start
at shared address `cur` and end with a sentinel entry whose pos is NP (the region size).
Each case loads the next entry's position before its FMAs (it feeds the next branch)
and the next value after them (into the register its FMAs just read), so no register
copies are needed between nonzeros.

usage: python gen_si_cases.py > si3x3_cases.inc
"""

TILES = [(4, 8)]


def block(ty, tx):
    ry_n, rx_n = ty + 2, tx + 2
    np_ = ry_n * rx_n
    na = ty * tx
    A = lambda oy, ox: f"%{oy * tx + ox}"
    W = lambda kh, kw: f"%{na + kh * 3 + kw}"
    I_CUR = f"%{na + 9}"
    L = []
    e = L.append
    e("{")
    e(".reg .b32 r_cur, r_ix;")
    e(".reg .f32 f_v;")
    e(f"mov.b32 r_cur, {I_CUR};")
    targets = ", ".join([f"P{p}_%=" for p in range(np_)] + ["D_%="])
    e(f"T_%=: .branchtargets {targets};")
    e("ld.volatile.shared.b32 r_ix, [r_cur];")
    e("ld.volatile.shared.f32 f_v, [r_cur+4];")
    e("N_%=:")
    e("add.u32 r_cur, r_cur, 8;")
    e("brx.idx.uni r_ix, T_%=;")
    for p in range(np_):
        ry, rx = divmod(p, rx_n)
        e(f"P{p}_%=:")
        e("ld.volatile.shared.b32 r_ix, [r_cur];")
        for kh in range(3):
            for kw in range(3):
                oy, ox = ry - kh, rx - kw
                if 0 <= oy < ty and 0 <= ox < tx:
                    e(f"fma.rn.f32 {A(oy, ox)}, {W(kh, kw)}, f_v, {A(oy, ox)};")
        e("ld.volatile.shared.f32 f_v, [r_cur+4];")
        e("bra.uni N_%=;")
    e("D_%=:")
    e("}")
    return "\\n\\t".join(L)


def emit(ty, tx):
    na = ty * tx
    outs = ", ".join(f'"+f"(acc[{i}])' for i in range(na))
    ins = ", ".join(f'"f"(wt[{t}])' for t in range(9))
    print(f"// tile {ty} x {tx}: region {ty + 2} x {tx + 2}")
    print("template <>")
    print(f"__device__ __forceinline__ void si_chan<{ty}, {tx}>(float (&acc)[{na}], const float (&wt)[9], uint32_t cur) {{")
    print(f'    asm volatile("{block(ty, tx)}"')
    print(f"                 : {outs}")
    print(f'                 : {ins}, "r"(cur)')
    print('                 : "memory");')
    print("}")
    print()


def blockp(ty, tx, pairs):
    """Lane = 2 * pairs filters: the accumulator of an output is `pairs` register pairs
    (f0, f1), (f2, f3), ..., a tap's weights the same number of pairs, the input value
    is broadcast: every FMA is an FFMA2, `pairs` of them per (nonzero, tap).

    Walks one channel block of a tile stream page in shared memory: entries {pos, value
    bits} in ascending position, closed by a link {NP or NP + 1, next channel}.  The next
    entry is loaded with one 64-bit shared load after a case's FMAs, into the registers
    it has finished with (no copies); both link kinds leave through D with the cursor
    past the link and the link's two words in (lx, ly).

    Measured alternatives (VGG16 layer 8, 90 % input zeros): entries that carry the next
    entry's position so a case knows its successor before its FMAs (+7 %: the shared
    load was not the limit), and a dispatch replicated at the end of every case so the
    jump-table lookup can start early (1.7x slower: ptxas gives every branch its own
    constant-bank table).  The limit is the indirect branch itself (~1 per 14-18 cycles
    per SM whatever the tile or occupancy), so the lever is FMAs per branch: pairs = 2
    (4 filters per lane) from K = 128."""
    ry_n, rx_n = ty + 2, tx + 2
    np_ = ry_n * rx_n
    na = ty * tx
    A = lambda oy, ox, h: f"%{(oy * tx + ox) * pairs + h}"
    W = lambda kh, kw, h: f"%{na * pairs + 3 + (kh * 3 + kw) * pairs + h}"
    CUR, LX, LY = f"%{na * pairs}", f"%{na * pairs + 1}", f"%{na * pairs + 2}"
    L = []
    e = L.append
    e("{")
    e(".reg .b32 r_ix, r_vb;")
    e(".reg .f32 f_v;")
    e(".reg .b64 d_vv;")
    targets = ", ".join([f"P{p}_%=" for p in range(np_)] + ["D_%=", "D_%="])
    e(f"T_%=: .branchtargets {targets};")
    e(f"ld.shared.v2.b32 {{r_ix, r_vb}}, [{CUR}];")
    e("mov.b32 f_v, r_vb;")
    e("N_%=:")
    e(f"add.u32 {CUR}, {CUR}, 8;")
    e("brx.idx.uni r_ix, T_%=;")
    for p in range(np_):
        ry, rx = divmod(p, rx_n)
        e(f"P{p}_%=:")
        e("mov.b64 d_vv, {f_v, f_v};")
        for kh in range(3):
            for kw in range(3):
                oy, ox = ry - kh, rx - kw
                if 0 <= oy < ty and 0 <= ox < tx:
                    for h in range(pairs):
                        e(f"fma.rn.f32x2 {A(oy, ox, h)}, d_vv, {W(kh, kw, h)}, {A(oy, ox, h)};")
        e(f"ld.shared.v2.b32 {{r_ix, r_vb}}, [{CUR}];")
        e("mov.b32 f_v, r_vb;")
        e("bra.uni N_%=;")
    e("D_%=:")
    e(f"mov.b32 {LX}, r_ix;")
    e(f"mov.b32 {LY}, r_vb;")
    e("}")
    return "\\n\\t".join(L)


def emitp(ty, tx, pairs):
    na = ty * tx
    outs = ", ".join([f'"+l"(acc[{i}])' for i in range(na * pairs)] + ['"+r"(cur)', '"=r"(lx)', '"=r"(ly)'])
    ins = ", ".join(f'"l"(wt[{t}])' for t in range(9 * pairs))
    print(f"// {2 * pairs} filters per lane, tile {ty} x {tx}: region {ty + 2} x {tx + 2}")
    print("template <>")
    print(f"__device__ __forceinline__ void si_chanp<{ty}, {tx}, {pairs}>(unsigned long long (&acc)[{na * pairs}],")
    print(f"        const unsigned long long (&wt)[{9 * pairs}], uint32_t &cur, int &lx, int &ly) {{")
    print(f'    asm volatile("{blockp(ty, tx, pairs)}"')
    print(f"                 : {outs}")
    print(f"                 : {ins}")
    print('                 : "memory");')
    print("}")
    print()


TILESP = [(4, 8, 1), (4, 4, 2)]


def main():
    print("// GENERATED by gen_si_cases.py -- do not edit by hand.")
    print("template <int TY, int TX>")
    print("__device__ __forceinline__ void si_chan(float (&acc)[TY * TX], const float (&wt)[9], uint32_t cur);")
    print()
    for ty, tx in TILES:
        emit(ty, tx)
    print("template <int TY, int TX, int PAIRS>")
    print("__device__ __forceinline__ void si_chanp(unsigned long long (&acc)[TY * TX * PAIRS],")
    print("        const unsigned long long (&wt)[9 * PAIRS], uint32_t &cur, int &lx, int &ly);")
    print()
    for ty, tx, pairs in TILESP:
        emitp(ty, tx, pairs)


if __name__ == "__main__":
    main()
