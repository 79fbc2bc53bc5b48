"""Seeded synthetic workload generator (inputs only — no convolution arithmetic).

This module is the ONE piece shared by the oracle side (``oracle/``, ``tests/``)
and the CUDA side (``paper_2005_04091_b200``, ``bench.py``).  It draws random
numbers and lays them out as the C-ABI's input format; it computes nothing the
method computes (no decode, no convolution, no pooling).

Recipe:

* PRNG: counter-based SplitMix64.  Element ``i`` of stream ``seed`` is
  ``mix64(seed + (i + 1) * 0x9E3779B97F4A7C15 mod 2^64)``, so any element can be
  regenerated on its own (used by sampled parity checks at full size).
* Float draw: ``f = (u >> 40) * 2^-23 - 1`` in [-1, 1); 24-bit grid, exactly
  representable in FP32 and never denormal.
* Weight positions (unstructured magnitude pruning stand-in, PAPER.md L383-387,
  Table 1): exactly ``nnz = round(d * F*C*K*K)`` positions, uniform
  without replacement over the whole (F, C*K*K) matrix — the ``nnz`` positions
  with the smallest 64-bit keys of stream ``seed(k, 0)``.  Per-row counts then
  vary (binomial-like), which exercises load balancing.
* Weight values: U[-1, 1) from stream ``seed(k, 1)`` at counter = flat position;
  an exact 0 is redrawn at counter ``pos + M*t`` (t = 1, 2, ...).
* Inputs: U[-1, 1) from stream ``seed(k, 2)`` at counter = flat NCHW index.
* Bias: U[-0.5, 0.5) from stream ``seed(k, 3)`` (the float draw halved).
* Integer mode (exact-arithmetic pin): weights in {+-1..+-4}, inputs in
  {-4..4}, bias in {-2..2}.
* Seeds: ``seed(k, stream) = 2005040910 + 10*k + stream`` (k = config 1..5).

The CSR layout produced is the C-ABI boundary format (include/spconv.h):
``rowptr[F+1]`` int32, ``colidx[nnz]`` int32 = ``(c*K + ky)*K + kx`` ascending per
row (flatten (F, C, K, K) -> (F, C*K*K), compress rows), and
``values[nnz]`` float32.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
SEED_BASE = 2005040910


def seed_of(k: int, stream: int) -> int:
    """Seed for config ``k`` (1..5) and stream (0 positions, 1 values, 2 input, 3 bias)."""
    return SEED_BASE + 10 * k + stream


def splitmix64(seed: int, counters: np.ndarray) -> np.ndarray:
    """Counter-based SplitMix64: element ``i`` -> mix64(seed + (i+1)*GAMMA)."""
    c = np.asarray(counters, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (c + np.uint64(1)) * GAMMA
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def unit_float(u: np.ndarray) -> np.ndarray:
    """u (uint64) -> float32 in [-1, 1) on a 2^-23 grid (exact in FP32)."""
    return ((u >> np.uint64(40)).astype(np.float64) * (2.0 ** -23) - 1.0).astype(np.float32)


def int_value(u: np.ndarray, lo: int, hi: int, nonzero: bool = False) -> np.ndarray:
    """u (uint64) -> integer-valued float32 uniform in [lo, hi] (optionally skipping 0)."""
    top = (u >> np.uint64(32)).astype(np.int64)
    if nonzero:
        span = hi - lo  # e.g. {-4..-1, 1..4} has 8 values for lo=-4, hi=4
        v = top % span + lo
        v = np.where(v >= 0, v + 1, v)
    else:
        v = top % (hi - lo + 1) + lo
    return v.astype(np.float32)


def nnz_for(F: int, C: int, K: int, density: float) -> int:
    """nnz = round(d * F*C*K*K) (round half up)."""
    return int(math.floor(density * F * C * K * K + 0.5))


@dataclass
class CSR:
    F: int
    C: int
    K: int
    rowptr: np.ndarray  # int32 [F+1]
    colidx: np.ndarray  # int32 [nnz]
    values: np.ndarray  # float32 [nnz]

    @property
    def nnz(self) -> int:
        return int(self.colidx.shape[0])


def make_csr(F: int, C: int, K: int, density: float, seed_pos: int, seed_val: int,
             integer: bool = False, skew: float = 0.0) -> CSR:
    """Random CSR filters with exactly round(d*F*C*K^2) nonzeros.

    ``skew`` > 0 selects the optional skewed-row mode: per-row keys are biased
    by a log-uniform per-row weight so row densities spread (LTH-like layers,
    PAPER.md L386).  ``skew = 0`` is uniform without replacement.
    """
    M = F * C * K * K
    nnz = nnz_for(F, C, K, density)
    keys = splitmix64(seed_pos, np.arange(M, dtype=np.uint64))
    if skew > 0.0:
        # per-row log-uniform weight in [e^-skew, e^skew]; key scaled down for heavy rows
        rowu = unit_float(splitmix64(seed_pos ^ 0x5DEECE66D, np.arange(F, dtype=np.uint64)))
        wrow = np.exp(skew * rowu.astype(np.float64))
        kf = (keys >> np.uint64(11)).astype(np.float64) / float(1 << 53)
        kf = kf ** (1.0 / np.repeat(wrow, C * K * K))
        order = np.argsort(kf, kind="stable")
    else:
        order = np.argsort(keys, kind="stable")
    pos = np.sort(order[:nnz]).astype(np.int64)
    CKK = C * K * K
    rows = pos // CKK
    cols = (pos % CKK).astype(np.int32)
    counts = np.bincount(rows, minlength=F)
    rowptr = np.zeros(F + 1, dtype=np.int32)
    rowptr[1:] = np.cumsum(counts)
    upos = pos.astype(np.uint64)
    if integer:
        vals = int_value(splitmix64(seed_val, upos), -4, 4, nonzero=True)
    else:
        vals = unit_float(splitmix64(seed_val, upos))
        t = 1
        while True:
            z = vals == 0.0
            if not z.any():
                break
            vals[z] = unit_float(splitmix64(seed_val, upos[z] + np.uint64(M * t)))
            t += 1
    return CSR(F, C, K, rowptr, cols, vals.astype(np.float32))


def make_input(shape, seed: int, integer: bool = False, chunk: int = 1 << 24,
               out: np.ndarray | None = None) -> np.ndarray:
    """NCHW float32 input; element i drawn from counter i of stream ``seed``."""
    n = int(np.prod(shape))
    if out is None:
        out = np.empty(n, dtype=np.float32)
    flat = out.reshape(-1)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        u = splitmix64(seed, np.arange(s, e, dtype=np.uint64))
        flat[s:e] = int_value(u, -4, 4) if integer else unit_float(u)
    return out.reshape(shape)


def input_at(seed: int, flat_index: np.ndarray, integer: bool = False) -> np.ndarray:
    """Regenerate individual input elements (counter-based)."""
    u = splitmix64(seed, np.asarray(flat_index, dtype=np.uint64))
    return int_value(u, -4, 4) if integer else unit_float(u)


def make_bias(F: int, seed: int, integer: bool = False) -> np.ndarray:
    u = splitmix64(seed, np.arange(F, dtype=np.uint64))
    if integer:
        return int_value(u, -2, 2)
    return (unit_float(u) * np.float32(0.5)).astype(np.float32)


@dataclass(frozen=True)
class LayerConfig:
    """One BASELINE.json workload."""
    k: int
    name: str
    N: int
    C: int
    H: int
    W: int
    F: int
    K: int
    stride: int
    pad: int
    density: float
    fused: bool
    bias: bool
    note: str = ""

    @property
    def Ho(self) -> int:
        return (self.H + 2 * self.pad - self.K) // self.stride + 1

    @property
    def Wo(self) -> int:
        return (self.W + 2 * self.pad - self.K) // self.stride + 1

    @property
    def nnz(self) -> int:
        return nnz_for(self.F, self.C, self.K, self.density)

    @property
    def useful_flops(self) -> int:
        """Useful FLOPs = 2 * nnz * N * Ho * Wo (SURVEY.md §8 notation)."""
        return 2 * self.nnz * self.N * self.Ho * self.Wo

    def with_batch(self, N: int) -> "LayerConfig":
        return LayerConfig(self.k, self.name, N, self.C, self.H, self.W, self.F, self.K,
                           self.stride, self.pad, self.density, self.fused, self.bias, self.note)

    def with_density(self, d: float) -> "LayerConfig":
        return LayerConfig(self.k, self.name, self.N, self.C, self.H, self.W, self.F, self.K,
                           self.stride, self.pad, d, self.fused, self.bias, self.note)


# BASELINE.json "configs" (pad 1 for the K=3 layers: reading G6 in DESIGN.md).
CONFIGS = {
    "c1": LayerConfig(1, "c1", 1, 16, 16, 16, 16, 3, 1, 1, 0.20, False, False,
                      "single sparse conv N=1 C=16 H=W=16 F=16 K=3 pad=1 80% sparsity"),
    "c2": LayerConfig(2, "c2", 32, 64, 56, 56, 64, 3, 1, 1, 0.20, False, False,
                      "ResNet-style layer N=32 C=F=64 H=W=56 K=3 80% sparsity, conv only"),
    "c3": LayerConfig(3, "c3", 32, 64, 56, 56, 64, 3, 1, 1, 0.10, True, True,
                      "same layer fused sparse conv+bias+ReLU+2x2 maxpool, 90% sparsity"),
    "c4_50": LayerConfig(4, "c4_50", 64, 256, 14, 14, 256, 3, 1, 1, 0.50, False, False,
                         "C=F=256 H=W=14 K=3 N=64, 50% sparsity"),
    "c4_80": LayerConfig(4, "c4_80", 64, 256, 14, 14, 256, 3, 1, 1, 0.20, False, False,
                         "C=F=256 H=W=14 K=3 N=64, 80% sparsity"),
    "c4_90": LayerConfig(4, "c4_90", 64, 256, 14, 14, 256, 3, 1, 1, 0.10, False, False,
                         "C=F=256 H=W=14 K=3 N=64, 90% sparsity"),
    "c4_95": LayerConfig(4, "c4_95", 64, 256, 14, 14, 256, 3, 1, 1, 0.05, False, False,
                         "C=F=256 H=W=14 K=3 N=64, 95% sparsity"),
    "c5": LayerConfig(5, "c5", 256, 128, 112, 112, 128, 3, 1, 1, 0.15, False, False,
                      "VGG-style C=F=128 H=W=112 K=3 85% sparsity N=256 batch-sharded"),
}


@dataclass
class Layer:
    cfg: LayerConfig
    csr: CSR
    bias: np.ndarray | None
    x: np.ndarray | None = field(default=None, repr=False)


def make_layer(cfg: LayerConfig, integer: bool = False, with_input: bool = True,
               skew: float = 0.0) -> Layer:
    """Filters, bias and (optionally) the input for config ``cfg``."""
    k = cfg.k
    csr = make_csr(cfg.F, cfg.C, cfg.K, cfg.density, seed_of(k, 0), seed_of(k, 1),
                   integer=integer, skew=skew)
    bias = make_bias(cfg.F, seed_of(k, 3), integer=integer) if cfg.bias else None
    x = make_input((cfg.N, cfg.C, cfg.H, cfg.W), seed_of(k, 2), integer=integer) if with_input else None
    return Layer(cfg, csr, bias, x)


# ---------------------------------------------------------------- NEXT-4: sparse multilayer LSTM
def lstm_seed(layer: int, stream: int) -> int:
    """Seeds of the LSTM workload: 2005040960 + 10*layer + stream (0 positions,
    1 values, 3 bias); the input uses stream 2 of layer 0."""
    return SEED_BASE + 50 + 10 * layer + stream


def make_lstm(L: int, D: int, H: int, density: float, T: int, B: int):
    """Per layer the CSR of the fused gate matrix [W | U] (4H x (D_l + H), gate rows i, f,
    g, o), bias [4H] and the input x [T, B, D].

    Positions uniform without replacement at ``density`` ("15% as a
    uniformly distributed density level"); values U[-1, 1) scaled by 1/sqrt(expected
    nonzeros per row) so the gate pre-activations stay O(1) (input recipe);
    bias U[-0.5, 0.5); inputs U[-1, 1)."""
    layers = []
    for l in range(L):
        Dl = D if l == 0 else H
        csr = make_csr(4 * H, Dl + H, 1, density, lstm_seed(l, 0), lstm_seed(l, 1))
        scale = np.float32(1.0 / math.sqrt(max(1.0, density * (Dl + H))))
        vals = (csr.values * scale).astype(np.float32)
        layers.append((csr.rowptr, csr.colidx, vals, make_bias(4 * H, lstm_seed(l, 3))))
    x = make_input((T, B, D), lstm_seed(0, 2))
    return layers, x
