"""Generate dispatch2_gen.inc: the tap dispatcher of kernel_pipe.cu (v2 kernel).

For one (row group, pipeline stage of input channels) a warp walks a
shared-memory stream of 8-byte entries {v, case of the NEXT entry} (the
segment starts with a lead entry holding the first case).  Every tap
case = r*9 + ky*3 + kx selects the FMAs of one CSR nonzero on the thread's
T x S output tile ("out[n][y][x] +=
coeff * in[...]"):

    acc[r][t][s] = fma(v, x[t+ky][s+kx], acc[r][t][s])   t < T, s < S

Accumulators and the (T+2) x (S+2) input window live in 64-bit register
pairs so that the even-kx cases issue packed fma.rn.f32x2 (FFMA2: T*S/2
instructions for T*S FMAs, per-component rounding identical to fmaf); kx = 1
needs the odd pairs (x1,x2),(x3,x4),..., which are not register pairs, and
issues T*S scalar FFMA.

Dispatch is "threaded code" through one brx.idx jump table, software-
pipelined: the case id of nonzero k+1 is already in a register when case k
starts, so the jump-table load for k+1 (an indexed constant load) is issued
at the top of case k and overlaps its FMAs; case k loads the case id of
entry k+2 early and, after its FMAs, the VALUE of entry k+1 straight into the
FMA operand register (its latency hides under the branch).  Long case bodies (T*S FMAs) are
what hide the jump latency (scripts/probes/dispatch_probe.cu measures it).

One walk covers all channels of a pipeline stage: case R*9 ("next channel")
advances the window pointer by k staged channels (k = the marker entry's value
field: channels without nonzeros for the group are skipped, not reloaded) and
reloads the window from shared memory, case R*9+1 ends the walk.

Run: python gen_dispatch2.py [out]  (build.py runs it when the output is stale).
"""
import os
import sys

# (R, T, S) variants instantiated by kernel_pipe.cu
VARIANTS = [(4, 4, 8), (4, 8, 4), (4, 4, 4), (2, 8, 4), (4, 7, 4), (2, 7, 4)]
MASK_VARIANTS = [(4, 8, 4)]
# dispatcher code variants (A/B via -DSPC_DISPATCH_VARIANT=v): 0 = round-1 walk,
# 1 = sp advanced in the case head (no write-after-read stall at the case end),
# 2 = 1 + a single brx.idx site (one jump table instead of one per case),
# 3 = 1 + the new sp forced before the loads, 4 = 3 + a single site,
# 5 = 3 + the next case id loaded (volatile) at the top of the case
DISPATCH_VARIANTS = [0, 1, 2, 3, 4, 5]
# Stream entries are 8 bytes {value (f32), case of the NEXT entry (u32)}: the value
# is loaded straight into the FMA operand at the end of a case (FFMA2 takes it as a
# broadcast .F32 operand), the next case id early -- no register copies.  (Measured
# on B200: 16-byte {v, v, case, 0} entries with one load and register copies were
# 2.3% slower on c2.)
ENT = 8


def gen(R: int, T: int, S: int, variant: int = 0) -> str:
    PAIRS = (S + 2) // 2  # window pairs per row
    SH = S // 2           # accumulator pairs per output row
    nacc = R * T * SH

    def A(r, t, h):
        return f"%{(r * T + t) * SH + h}"

    XBASE = nacc + 1  # operand index of the first window pair (after the pointer output)

    def X(i, j):
        return f"%{XBASE + i * PAIRS + j}"

    def head():
        # case id of entry k+1 (it came with entry k): its jump-table load overlaps
        # this case's FMAs.  variant >= 1: sp advances here, one branch away from the
        # last load that read it (advancing it after that load stalled the end of
        # every case on the load's register read, a write-after-read hazard)
        out = ["mov.b32 %%cn, %%cx;"]
        if variant >= 1:
            # the stride comes in a register (SPC2_ENT_REG): with an immediate, ptxas
            # folds the add into the loads' offsets and copies the new sp back after
            # the last load -- the very hazard this avoids
            out.append(f"add.u32 %%sp, %%sp, {ENTR};")
            if variant >= 3:
                # a no-op mask (entries are 8-byte aligned) that ptxas cannot fold into
                # the loads' address: the new sp must exist before them
                out.append("and.b32 %%sp, %%sp, -8;")
            if variant >= 5:
                # the case id of entry k+2 at the top (volatile: not merged with the
                # value load at the end into one 64-bit load, which would put the
                # load's latency in front of the next case's jump-table load)
                out.append("ld.volatile.shared.u32 %%cx, [%%sp+4];")
        return out

    def tail():
        # after the FMAs, entry k+1 = {v, case of k+2}: the value lands straight in
        # the operand register; sp -> entry k+2
        if variant >= 5:
            out = ["ld.shared.f32 %%vf, [%%sp];"]
        elif variant >= 1:
            out = ["ld.shared.f32 %%vf, [%%sp];",
                   "ld.shared.u32 %%cx, [%%sp+4];"]
        else:
            out = ["ld.shared.f32 %%vf, [%%sp];",
                   "ld.shared.u32 %%cx, [%%sp+4];",
                   f"add.u32 %%sp, %%sp, {ENT};"]
        if variant in (2, 4):
            # one dispatch site: a single jump table stays in the constant cache
            out.append(f"bra.uni $D{tag}_X;")
        else:
            out.append(f"brx.idx.uni %%cn, $D{tag}_T;")
        return out

    P = f"%{nacc}"  # u32 shared-memory stream address, in/out
    WP = f"%{nacc + 1 + (T + 2) * PAIRS}"  # u32 window address (in/out)
    CHS = f"%{nacc + 2 + (T + 2) * PAIRS}"  # channel stride in bytes (in)
    ROWB = f"%{nacc + 3 + (T + 2) * PAIRS}"  # row stride in bytes (in)
    ENTR = f"%{nacc + 4 + (T + 2) * PAIRS}"  # entry stride in bytes (in; == ENT)
    ncase = R * 9
    tag = f"R{R}T{T}S{S}"
    L = []
    L.append("{")
    L.append(".reg .b64 %%va;")  # (v, v): the FFMA2 operand (ptxas folds it into a .F32 broadcast)
    L.append(".reg .f32 %%vf;")  # the current entry's value
    L.append(".reg .b32 %%cn, %%cx, %%sp, %%wa;")
    L.append(".reg .f32 " + ", ".join(f"%%a{i}" for i in range(S)) + ", "
             + ", ".join(f"%%x{i}" for i in range(S + 2)) + ";")
    # P -> a lead entry whose case field is the first entry's case (the segment's
    # header entry, or a "next channel" marker when a walk starts mid-stage)
    L.append(f"mov.b32 %%sp, {P};")
    L.append("ld.shared.u32 %%cn, [%%sp+4];")
    L.append(f"ld.shared.f32 %%vf, [%%sp+{ENT}];")
    L.append(f"ld.shared.u32 %%cx, [%%sp+{ENT + 4}];")
    # variant 0: sp -> entry k+1 on entry to case k; variant >= 1: sp -> entry k
    # (the case head advances it)
    L.append(f"add.u32 %%sp, %%sp, {2 * ENT if variant == 0 else ENT};")
    L.append(f"$D{tag}_T: .branchtargets " + ", ".join(f"$D{tag}_{i}" for i in range(ncase + 2)) + ";")
    if variant in (2, 4):
        L.append(f"$D{tag}_X:")
    L.append(f"brx.idx.uni %%cn, $D{tag}_T;")
    for i in range(ncase):
        # tap-major case numbering: case = (ky*3 + kx)*R + r
        r, ky, kx = i % R, (i // R) // 3, (i // R) % 3
        L.append(f"$D{tag}_{i}:")
        L += head()
        if kx != 1:
            L.append("mov.b64 %%va, {%%vf, %%vf};")
            for t in range(T):
                for h in range(SH):
                    L.append(f"fma.rn.f32x2 {A(r, t, h)}, %%va, {X(t + ky, h + kx // 2)}, {A(r, t, h)};")
        else:
            for t in range(T):
                row = t + ky
                for j in range(PAIRS):
                    L.append(f"mov.b64 {{%%x{2 * j}, %%x{2 * j + 1}}}, {X(row, j)};")
                for h in range(SH):
                    L.append(f"mov.b64 {{%%a{2 * h}, %%a{2 * h + 1}}}, {A(r, t, h)};")
                for s in range(S):
                    L.append(f"fma.rn.f32 %%a{s}, %%vf, %%x{s + 1}, %%a{s};")
                for h in range(SH):
                    L.append(f"mov.b64 {A(r, t, h)}, {{%%a{2 * h}, %%a{2 * h + 1}}};")
        L += tail()
    # next channel: advance the window and reload it (T+2 rows of PAIRS pairs)
    L.append(f"$D{tag}_{ncase}:")
    L += head()
    # the marker's value field holds k >= 1, the channels to advance (runs of channels
    # without nonzeros for this group are skipped in one step)
    L.append("mov.b32 %%wa, %%vf;")
    L.append(f"mad.lo.u32 {WP}, %%wa, {CHS}, {WP};")
    L.append(f"mov.b32 %%wa, {WP};")
    for i in range(T + 2):
        j = 0
        while j + 1 < PAIRS:
            L.append(f"ld.shared.v2.b64 {{{X(i, j)}, {X(i, j + 1)}}}, [%%wa+{8 * j}];")
            j += 2
        if j < PAIRS:
            L.append(f"ld.shared.b64 {X(i, j)}, [%%wa+{8 * j}];")
        if i + 1 < T + 2:
            L.append(f"add.u32 %%wa, %%wa, {ROWB};")
    L += tail()
    L.append(f"$D{tag}_{ncase + 1}:")
    if variant >= 1:
        L.append(f"add.u32 %%sp, %%sp, {ENTR};")
    L.append(f"mov.b32 {P}, %%sp;")
    L.append("}")
    asm = "\\n\\t".join(L)
    outs = ", ".join(f'"+l"(acc[{r}][{t}][{h}])' for r in range(R) for t in range(T) for h in range(SH))
    xws = ", ".join(f'"+l"(xw[{i}][{j}])' for i in range(T + 2) for j in range(PAIRS))
    return (f"#define SPC2_DISPATCH_{tag}(acc, xw, sp, wp, chs, rowb) \\\n"
            f"    asm volatile(\"{asm}\" \\\n"
            f"                 : {outs}, \"+r\"(sp), {xws}, \"+r\"(wp) \\\n"
            f"                 : \"r\"(chs), \"r\"(rowb), \"r\"(SPC2_ENT_REG) \\\n"
            f"                 : \"memory\")\n")


def gen_mask(R: int, T: int, S: int) -> str:
    """Mask walk for one channel (the default dispatcher, see kernel_pipe.cu).

    Operands: accumulator pairs (in/out), window pairs (in), the channel's 9R-bit
    tap x row mask (in), the smem address of the channel's DENSE value block (9R
    (v, v) pairs, zeros for absent taps; in) and the tap-0 values already loaded
    (R pairs, in/out: on exit they hold the NEXT channel's tap-0 values).

    Straight-line code over the 9R (tap, row) blocks in tap-major, row-minor
    order.  The values of tap t+1 are requested at the top of tap t into the other
    of two register sets (tap parity is static, so no copies); a tap with no row is
    skipped with one branch, a row without the tap with one more.  Branch
    conditions go through vote.sync so ptxas knows they are warp-uniform.
    """
    PAIRS = (S + 2) // 2
    SH = S // 2
    nacc = R * T * SH

    def A(r, t, h):
        return f"%{(r * T + t) * SH + h}"

    V0 = nacc              # first of R in/out value pairs (tap-0 set)
    XB = nacc + R

    def X(i, j):
        return f"%{XB + i * PAIRS + j}"

    M = f"%{XB + (T + 2) * PAIRS}"      # 64-bit mask (in)
    VB = f"%{XB + (T + 2) * PAIRS + 1}"  # u32 smem address of the dense values (in)
    tag = f"M{R}T{T}S{S}"
    # value registers: set 0 = the in/out operands, set 1 = locals
    def VAL(tap, r):
        return f"%{V0 + r}" if tap % 2 == 0 else f"%%w{r}"

    L = ["{", ".reg .pred %%p, %%q;", ".reg .b64 " + ", ".join(f"%%w{r}" for r in range(R)) + ";",
         ".reg .b32 %%mlo, %%mhi, %%mw, %%bt;",
         ".reg .f32 %%v1, %%vd, " + ", ".join(f"%%a{i}" for i in range(S)) + ", "
         + ", ".join(f"%%x{i}" for i in range(S + 2)) + ";",
         f"mov.b64 {{%%mlo, %%mhi}}, {M};"]

    def load_tap(tap):  # values of `tap` into its set (tap 9 = next channel's tap 0)
        out = []
        off = tap * R * 8
        regs = [VAL(tap, r) for r in range(R)]
        for r in range(0, R, 2):
            out.append(f"ld.shared.v2.b64 {{{regs[r]}, {regs[r + 1]}}}, [{VB}+{off + 8 * r}];")
        return out

    for tap in range(9):
        ky, kx = tap // 3, tap % 3
        L += load_tap(tap + 1)   # prefetch the next tap's values (tap 9 -> next channel's tap 0)
        lo_bit = tap * R
        if lo_bit + R <= 32:
            word, sh = "%%mlo", lo_bit
        elif lo_bit >= 32:
            word, sh = "%%mhi", lo_bit - 32
        else:
            word, sh = None, 0
        if word is not None:
            L.append(f"and.b32 %%mw, {word}, {((1 << R) - 1) << sh};")
        else:
            L.append(f"shf.r.clamp.b32 %%mw, %%mlo, %%mhi, {lo_bit};")
            L.append(f"and.b32 %%mw, %%mw, {(1 << R) - 1};")
        L.append("setp.eq.u32 %%p, %%mw, 0;")
        L.append(f"@%%p bra.uni $K{tag}_t{tap};")
        for r in range(R):
            L.append(f"and.b32 %%bt, %%mw, {1 << (sh + r)};")
            L.append("setp.eq.u32 %%p, %%bt, 0;")
            L.append(f"@%%p bra.uni $K{tag}_t{tap}r{r};")
            v = VAL(tap, r)
            if kx != 1:
                for t in range(T):
                    for h in range(SH):
                        L.append(f"fma.rn.f32x2 {A(r, t, h)}, {v}, {X(t + ky, h + kx // 2)}, {A(r, t, h)};")
            else:
                L.append(f"mov.b64 {{%%v1, %%vd}}, {v};")
                for t in range(T):
                    row = t + ky
                    for j in range(PAIRS):
                        L.append(f"mov.b64 {{%%x{2 * j}, %%x{2 * j + 1}}}, {X(row, j)};")
                    for h in range(SH):
                        L.append(f"mov.b64 {{%%a{2 * h}, %%a{2 * h + 1}}}, {A(r, t, h)};")
                    for s_ in range(S):
                        L.append(f"fma.rn.f32 %%a{s_}, %%v1, %%x{s_ + 1}, %%a{s_};")
                    for h in range(SH):
                        L.append(f"mov.b64 {A(r, t, h)}, {{%%a{2 * h}, %%a{2 * h + 1}}};")
            L.append(f"$K{tag}_t{tap}r{r}:")
        L.append(f"$K{tag}_t{tap}:")
    # tap 9 (odd) loaded into %%w: hand the next channel's tap-0 values back in set 0
    for r in range(R):
        L.append(f"mov.b64 %{V0 + r}, %%w{r};")
    L.append("}")
    asm = "\\n\\t".join(L)
    outs = ", ".join(f'"+l"(acc[{r}][{t}][{h}])' for r in range(R) for t in range(T) for h in range(SH))
    vals = ", ".join(f'"+l"(v0[{r}])' for r in range(R))
    ins = ", ".join(f'"l"(xw[{i}][{j}])' for i in range(T + 2) for j in range(PAIRS))
    return (f"#define SPC2_MASKWALK_{tag}(acc, v0, xw, m, vb) \\\n"
            f"    asm volatile(\"{asm}\" \\\n"
            f"                 : {outs}, {vals} \\\n"
            f"                 : {ins}, \"l\"(m), \"r\"(vb) \\\n"
            f"                 : \"memory\")\n")


def main(out_path: str) -> None:
    text = ["// GENERATED by gen_dispatch2.py — do not edit.\n"]
    text.append("#ifndef SPC_DISPATCH_VARIANT\n#define SPC_DISPATCH_VARIANT 3\n#endif\n")
    text.append(f"// the stream entry stride ({ENT}) as a register the compiler cannot fold\n"
                f"#ifndef SPC2_ENT_REG\n#define SPC2_ENT_REG {ENT}u\n#endif\n")
    for v in DISPATCH_VARIANTS:
        text.append(f"#if SPC_DISPATCH_VARIANT == {v}\n")
        for R, T, S in VARIANTS:
            text.append(f"// R={R} rows, thread tile T={T} x S={S}, window {T + 2} x {S + 2} as 64-bit pairs.\n")
            text.append(gen(R, T, S, v))
        text.append("#endif\n")
    for R, T, S in MASK_VARIANTS:
        text.append(f"// mask walk: R={R} rows, thread tile T={T} x S={S}.\n")
        text.append(gen_mask(R, T, S))
    tmp = out_path + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(text))
    os.replace(tmp, out_path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else
         os.path.join(os.path.dirname(os.path.abspath(__file__)), "dispatch2_gen.inc"))
