"""Per-CTA end-time analysis of SPCONV_PIPE_TRACE dumps (persistent pipe kernel).

usage: trace_ab.py TRACE_NORMAL TRACE_REVERSED
Tells whether slow CTAs follow the work (content imbalance) or the CTA/SM slot."""
import sys
import numpy as np


def load(path):
    out = []
    for blk in open(path).read().split("--"):
        rows = [l.split() for l in blk.strip().splitlines()]
        if len(rows) == 148:
            out.append(np.array([[int(x) for x in r] for r in rows]))
    return out


a, b = load(sys.argv[1]), load(sys.argv[2])
ea = np.mean([t[:, 4] for t in a], 0) / 1e3     # by CTA index (= work index)
eb = np.mean([t[:, 4] for t in b], 0) / 1e3     # by CTA index; work index = 147 - b
eb_work = eb[::-1]
print("normal  end min/med/max %.1f %.1f %.1f" % (ea.min(), np.median(ea), ea.max()))
print("reverse end min/med/max %.1f %.1f %.1f" % (eb.min(), np.median(eb), eb.max()))
print("corr(by work index)  %.3f" % np.corrcoef(ea, eb_work)[0, 1])
print("corr(by CTA/SM slot) %.3f" % np.corrcoef(ea, eb)[0, 1])
