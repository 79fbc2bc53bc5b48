"""Per-CTA end-time analysis of SPCONV_PIPE_TRACE dumps (kernel_pipe.cu debug trace:
blockIdx, SM, start, head parked, end, tail wait begin/end [ns], work index).

    python scripts/sk_trace_fit.py trace.txt [units C]

Prints the spread of CTA end times (the kernel ends with the slowest CTA), the mean
end by work-index quarter (a trend that follows the arrival ticket, not the work, is
hardware), and -- for the uniform split -- a least-squares fit of the end time on the
range structure (unit epilogues, head, tail), which is what sk_split's item costs
model."""
import sys

import numpy as np


def load(path):
    rows = [l.split() for l in open(path) if not l.startswith("--")]
    rows = [list(map(float, r)) for r in rows if len(r) == 8]
    G = int(max(r[0] for r in rows)) + 1
    return np.array(rows).reshape(-1, G, 8), G


def main():
    path = sys.argv[1]
    U = int(sys.argv[2]) if len(sys.argv) > 2 else 224
    C = int(sys.argv[3]) if len(sys.argv) > 3 else 64
    T, G = load(path)
    E = np.zeros(G)
    for blk in T:
        for r in blk:
            E[int(r[7])] += r[4] / len(T)
    print(f"{path}: {len(T)} launches, {G} CTAs")
    print(f"  mean end per work index: min {E.min():.0f} median {np.median(E):.0f} max {E.max():.0f} ns "
          f"(max - median {E.max() - np.median(E):.0f})")
    q = [E[i * G // 4:(i + 1) * G // 4].mean() for i in range(4)]
    print("  by work-index quarter:", " ".join(f"{v:.0f}" for v in q))
    X = []
    for b in range(G):
        s0, e0 = U * C * b // G, U * C * (b + 1) // G
        X.append([1.0, e0 // C - s0 // C, float(e0 % C > 0), float(s0 % C > 0)])
    x = np.linalg.lstsq(np.array(X), E, rcond=None)[0]
    print(f"  uniform-split fit: end = {x[0]:.0f} + {x[1]:.0f}*unit_epilogues + {x[2]:.0f}*head "
          f"+ {x[3]:.0f}*tail ns")


if __name__ == "__main__":
    main()
