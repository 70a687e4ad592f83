"""Generate sf3x3_dispatch.inc: the nonzero-dispatch loop of the fast sparse-filter
kernel for one staged chunk of input channels, as one inline-PTX block with a real
jump table.

Per chunk the lane walks a warp-uniform entry list: for each channel, the entries
(index = kl*9 + kh*3 + kw, value) of its filter group and a sentinel slot.  A jump
table (`brx.idx`) sends each entry to code that applies it to the lane's 4x4 output
tile of filter kl with statically named registers.  The channel's last entry carries
index + KT*9: its variant applies the entry and falls straight into the channel
transition (skip the sentinel slot, advance the patch pointer, reload the 6x6 input
patch, stop after the chunk's last channel) -- no extra dispatch per channel.  An
empty channel's sentinel slot carries 2*KT*9 and, in its value field, the length of the
run of empty channels it starts (bits 0-15): one dispatch skips the whole run.  A
transition loads only the patch rows the next channel's nonzeros touch: the row mask
travels in the value field of the previous channel's sentinel slot (or bits 16-21 of
an empty slot's value).  Why PTX: a
C++ switch becomes a 6-level compare tree and spills; this is one indirect branch per
nonzero and no per-channel call overhead.

Arithmetic: accumulators and the patch are held as 64-bit register pairs
(two adjacent columns).  Taps with kw in {0, 2} read column-aligned pairs and run as
8 FFMA2 (fma.rn.f32x2: two FP32 FMAs per instruction, same FMA-pipe rate, half the
issue slots); kw = 1 straddles the pairs and runs as 16 scalar FFMA on the halves.
The next entry is loaded at the top of each case (overlapping its FMAs).

Measured alternatives (tools/brx_bench.cu, B200): a 7-level compare-and-branch tree
instead of brx.idx is ~60 cycles/nonzero slower; replicating the dispatch at the end of
every case (no jump back to N_) is ~20% slower; loading the next entry before the BRX
instead of inside the case is ~3% slower.

Operands (all via the C++ wrapper sf3x3_chunk below; NA = 8*KT):
  %0..%NA-1     acc pairs  acc2[kl][py][h]  (kl*8 + py*2 + h), h=0: cols 0,1  h=1: cols 2,3
  next 18       patch pairs pt2[r][h]        (r*3 + h),         h: cols 2h, 2h+1
  then          entry cursor, patch cursor (shared addresses), channels left in the chunk,
                channel pitch of a staged box in bytes (register), row pitch in bytes
                (immediate, template parameter ROW_BYTES)

Run: python gen_sf3x3_dispatch.py > sf3x3_dispatch.inc
"""

TILE, PATCH = 4, 6




def load_patch(e, P, PP, RB, mask=None):
    # RB: the row pitch operand (an immediate; PTX folds the constant expression).
    # mask: register with one bit per patch row the channel's nonzeros touch (rows
    # kh..kh+3 of each); rows outside it keep the previous channel's values, which no
    # entry of this channel reads -- fewer shared-memory wavefronts on sparse channels.
    for r in range(PATCH):
        if mask is None:
            e(f"ld.shared.v2.b64 {{{P(r, 0)}, {P(r, 1)}}}, [{PP}+{RB}*{r}];")
            e(f"ld.shared.b64 {P(r, 2)}, [{PP}+{RB}*{r}+16];")
        else:
            e(f"and.b32 r_t, {mask}, {1 << r};")
            e(f"setp.ne.u32 q_r, r_t, 0;")
            e(f"@q_r ld.shared.v2.b64 {{{P(r, 0)}, {P(r, 1)}}}, [{PP}+{RB}*{r}];")
            e(f"@q_r ld.shared.b64 {P(r, 2)}, [{PP}+{RB}*{r}+16];")


def block(KT: int) -> str:
    NA = KT * 8                                              # acc pair operands
    A = lambda kl, py, h: f"%{kl * 8 + py * 2 + h}"          # acc pair
    P = lambda r, h: f"%{NA + r * 3 + h}"                    # patch pair
    # cursor, patch pointer and channel count arrive as plain inputs and are copied to
    # block-local registers: with read-write ("+r") operands ptxas wrapped the whole
    # dispatch loop in a per-nonzero convergence barrier (BSSY/BSYNC + an extra branch)
    # whenever the cursor was not a simple induction variable of the caller's loop
    I_CUR, I_PP, I_CNT, CHS, RB = (f"%{NA + 18 + i}" for i in range(5))
    CUR, PP, CNT = "r_cur", "r_pp", "r_cnt"
    NC = KT * 9
    L = []
    e = L.append
    e("{")
    e(".reg .pred p_end, q_r;")
    e(".reg .b32 r_t, r_m;")
    e(".reg .b32 r_ix, r_i1, r_v1, r_a, r_b, r_c, r_d, r_e, r_f;")
    e(".reg .b32 r_cur, r_pp, r_cnt;")
    e(f"mov.b32 r_cur, {I_CUR};")
    e(f"mov.b32 r_pp, {I_PP};")
    e(f"mov.b32 r_cnt, {I_CNT};")
    e(".reg .f32 f_v;")
    e(".reg .b64 d_vv;")
    # targets: 0..NC-1 entry, NC..2NC-1 channel-last entry, 2NC empty channel
    targets = ", ".join([f"C{i}_%=" for i in range(NC)] + [f"X{i}_%=" for i in range(NC)] + ["E_%="])
    e(f"T_%=: .branchtargets {targets};")
    load_patch(e, P, PP, RB)
    e(f"ld.shared.v2.b32 {{r_i1, r_v1}}, [{CUR}];")
    e(f"add.u32 {CUR}, {CUR}, 8;")
    e("N_%=:")
    e("mov.b32 f_v, r_v1;")
    e("mov.b32 r_ix, r_i1;")
    e("mov.b64 d_vv, {r_v1, r_v1};")
    e("brx.idx.uni r_ix, T_%=;")

    def prefetch():
        # the next entry is loaded at the top of each case, so the load overlaps the case's
        # FMAs (ptxas makes BRX wait on every outstanding scoreboard)
        e(f"ld.shared.v2.b32 {{r_i1, r_v1}}, [{CUR}];")
        e(f"add.u32 {CUR}, {CUR}, 8;")

    def fmas(kl, tap):
        kh, kw = divmod(tap, 3)
        for py in range(TILE):
            r = py + kh
            if kw in (0, 2):
                for h in range(2):
                    src = P(r, h + kw // 2)
                    a = A(kl, py, h)
                    e(f"fma.rn.f32x2 {a}, d_vv, {src}, {a};")
            else:
                # window cols 1..4 = hi(pair0), lo(pair1), hi(pair1), lo(pair2)
                e(f"mov.b64 {{r_a, r_b}}, {P(r, 0)};")
                e(f"mov.b64 {{r_c, r_d}}, {P(r, 1)};")
                e(f"mov.b64 {{r_e, r_f}}, {P(r, 2)};")
                for h in range(2):
                    lo_src, hi_src = (("r_b", "r_c"), ("r_d", "r_e"))[h]
                    a = A(kl, py, h)
                    e("{ .reg .f32 x, y;")
                    e(f"mov.b64 {{x, y}}, {a};")
                    e(f"fma.rn.f32 x, f_v, {lo_src}, x;")
                    e(f"fma.rn.f32 y, f_v, {hi_src}, y;")
                    e(f"mov.b64 {a}, {{x, y}};")
                    e("}")

    for kl in range(KT):
        for tap in range(9):
            e(f"C{kl * 9 + tap}_%=:")
            prefetch()
            fmas(kl, tap)
            e("bra.uni N_%=;")
    for kl in range(KT):
        for tap in range(9):
            e(f"X{kl * 9 + tap}_%=:")
            prefetch()
            fmas(kl, tap)
            e("bra.uni S_%=;")
    # channel-last entry: the prefetched slot was the segment's sentinel; skip it
    e("S_%=:")
    e(f"sub.u32 {CNT}, {CNT}, 1;")
    e(f"setp.eq.u32 p_end, {CNT}, 0;")
    e("@p_end bra.uni D_%=;")
    e(f"add.u32 {PP}, {PP}, {CHS};")
    e("mov.b32 r_m, r_v1;")  # the sentinel slot's value: the next channel's row mask
    load_patch(e, P, PP, RB, "r_m")
    e(f"ld.shared.v2.b32 {{r_i1, r_v1}}, [{CUR}];")
    e(f"add.u32 {CUR}, {CUR}, 8;")
    e("bra.uni N_%=;")
    # empty channel: the prefetched entry already belongs to the next channel
    # empty channels: the slot's value field holds the length of the run of empty
    # channels starting here (>= 1); skip the whole run (clipped to the chunk) with one
    # dispatch and one patch load for the next non-empty channel
    e("E_%=:")
    e("mov.b32 r_ix, f_v;")
    e("shr.u32 r_m, r_ix, 16;")  # the next non-empty channel's row mask
    e("and.b32 r_ix, r_ix, 65535;")
    e(f"min.u32 r_ix, r_ix, {CNT};")
    e(f"sub.u32 {CNT}, {CNT}, r_ix;")
    e(f"setp.eq.u32 p_end, {CNT}, 0;")
    e("@p_end bra.uni D_%=;")
    e(f"mad.lo.u32 {PP}, r_ix, {CHS}, {PP};")
    e("add.u32 r_ix, r_ix, -1;")
    e(f"mad.lo.u32 {CUR}, r_ix, 8, {CUR};")
    e(f"ld.shared.v2.b32 {{r_i1, r_v1}}, [{CUR}];")
    e(f"add.u32 {CUR}, {CUR}, 8;")
    load_patch(e, P, PP, RB, "r_m")
    e("bra.uni N_%=;")
    e("D_%=:")
    e("}")
    return "\\n\\t".join(L)


def emit(KT: int) -> None:
    outs = ", ".join(f'"+l"(acc2[{kl}][{py}][{h}])' for kl in range(KT) for py in range(TILE) for h in range(2))
    pts = ", ".join(f'"=l"(pt2[{r}][{h}])' for r in range(PATCH) for h in range(3))
    print("template <int ROW_BYTES>")
    print(f"__device__ __forceinline__ void sf3x3_chunk(unsigned long long (&acc2)[{KT}][4][2],")
    print("                                            uint32_t cur, uint32_t patch, uint32_t n_ch,")
    print("                                            uint32_t ch_bytes) {")
    print("    unsigned long long pt2[6][3];")
    print(f'    asm volatile("{block(KT)}"')
    print(f"                 : {outs},")
    print(f"                   {pts}")
    print('                 : "r"(cur), "r"(patch), "r"(n_ch), "r"(ch_bytes), "n"(ROW_BYTES)')
    print('                 : "memory");')
    print("}")
    print()


def main():
    print("// GENERATED by gen_sf3x3_dispatch.py -- do not edit by hand.")
    print("// One staged chunk of input channels of the fast sparse-filter kernel (overloads")
    print("// for KT = 1, 2, 4 and 8 filters per warp); see the generator for the protocol.")
    for kt in (1, 2, 4, 8):
        emit(kt)


if __name__ == "__main__":
    main()
