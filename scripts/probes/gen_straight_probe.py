"""Probe generator: straight-line FFMA2 'JIT' code (values as immediates) to
measure how instruction-stream size and per-warp stream divergence affect FP32
FMA throughput on B200.  Emits a standalone PTX kernel `probe`.

usage: gen_straight_probe.py OUT.ptx M NSTREAMS KX1FRAC
  M        cases per stream (one case = one nonzero: 16 FFMA2 or 32 FFMA)
  NSTREAMS distinct code streams (warp w runs stream w % NSTREAMS when mode=1)
"""
import random, struct, sys

out, M, NS, kx1 = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
R, T, SH = 4, 4, 4           # 4 rows x (4 tile rows x 8 cols = 4 x 4 pairs)
rnd = random.Random(7)
L = []
A = lambda r, t, h: f"%a{(r * T + t) * SH + h}"
X = lambda row, j: f"%w{row * 5 + j}"      # 6 rows x 5 pairs
def f32hex(x):
    return "0f%08X" % struct.unpack("<I", struct.pack("<f", x))[0]
L += [".version 8.7", ".target sm_100a", ".address_size 64",
      ".visible .entry probe(.param .u64 out, .param .u32 reps, .param .u32 mode)",
      ".maxntid 256, 1, 1", "{",
      ".reg .b64 %a<64>;", ".reg .b64 %w<30>;", ".reg .b64 %v;", ".reg .b32 %r<16>;",
      ".reg .pred %p<4>;", ".reg .b64 %rd<8>;", ".reg .f32 %f<70>;",
      ".shared .align 16 .b8 win[24576];"]
for i in range(64):
    L.append(f"mov.b64 %a{i}, 0;")
L += ["mov.u32 %r0, %tid.x;", "and.b32 %r1, %r0, 31;", "shr.u32 %r2, %r0, 5;",
      "mul.lo.u32 %r3, %r1, 16;", "mov.u32 %r4, win;", "add.u32 %r4, %r4, %r3;",  # lane base
      "ld.param.u32 %r5, [reps];", "ld.param.u32 %r6, [mode];",
      "mov.u32 %r7, 0;", "setp.eq.u32 %p1, %r6, 0;",
      f"rem.u32 %r8, %r2, {NS};", "selp.u32 %r8, 0, %r8, %p1;"]
for i in range(30):
    L.append(f"ld.shared.v2.b64 {{{X(i // 5, i % 5)}, %v}}, [%r4+{(i * 16) % 8192}];")
L.append("LOOP:")
for s in range(NS):
    L.append(f"setp.eq.u32 %p2, %r8, {s};")
    L.append(f"@%p2 bra S{s};")
L.append("bra END;")
for s in range(NS):
    L.append(f"S{s}:")
    for k in range(M):
        if k % 7 == 6:   # channel change: reload the window (15 x 16-byte loads)
            for i in range(15):
                off = (rnd.randrange(0, 512) * 512 + i * 16) % 24576 & ~15
                L.append(f"ld.shared.v2.b64 {{{X((2*i) // 5, (2*i) % 5)}, {X((2*i+1) // 5, (2*i+1) % 5)}}}, [%r4+{off % 8192}];")
        r, ky = rnd.randrange(R), rnd.randrange(3)
        kx = 1 if rnd.random() < kx1 else rnd.choice((0, 2))
        v = rnd.uniform(-1, 1)
        if kx != 1:
            h = f32hex(v)[2:]
            L.append(f"mov.b64 %v, 0x{h}{h};")
            for t in range(T):
                for hh in range(SH):
                    L.append(f"fma.rn.f32x2 {A(r, t, hh)}, %v, {X(t + ky, hh + kx // 2)}, {A(r, t, hh)};")
        else:
            for t in range(T):
                for hh in range(SH):
                    # scalar FFMA on odd pairs: unpack is register renaming in SASS
                    L.append(f"{{ .reg .f32 %lo, %hi, %x0, %x1, %x2, %x3; mov.b64 {{%lo, %hi}}, {A(r, t, hh)};"
                             f" mov.b64 {{%x0, %x1}}, {X(t + ky, hh)}; mov.b64 {{%x2, %x3}}, {X(t + ky, hh + 1)};"
                             f" fma.rn.f32 %lo, {f32hex(v)}, %x1, %lo; fma.rn.f32 %hi, {f32hex(v)}, %x2, %hi;"
                             f" mov.b64 {A(r, t, hh)}, {{%lo, %hi}}; }}")
    L.append("bra NEXT;")
L += ["NEXT:", "add.u32 %r7, %r7, 1;", "setp.lt.u32 %p3, %r7, %r5;", "@%p3 bra LOOP;", "END:"]
# reduce and store
L.append("mov.f32 %f0, 0f00000000;")
for i in range(64):
    L.append(f"{{ .reg .f32 %lo, %hi; mov.b64 {{%lo, %hi}}, %a{i}; add.f32 %f0, %f0, %lo; add.f32 %f0, %f0, %hi; }}")
L += ["ld.param.u64 %rd0, [out];", "mov.u32 %r9, %ctaid.x;", "mad.lo.u32 %r10, %r9, 256, %r0;",
      "mul.wide.u32 %rd1, %r10, 4;", "add.u64 %rd2, %rd0, %rd1;", "st.global.f32 [%rd2], %f0;", "ret;", "}"]
open(out, "w").write("\n".join(L) + "\n")
