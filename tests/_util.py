"""Test-side helpers (pins written independently of oracle/ and of the CUDA path)."""
from __future__ import annotations

import ctypes
import json
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")
_BRUTE_SRC = os.path.join(HERE, "pins", "brute_dense.c")
_BRUTE_LIB = os.path.join(HERE, "pins", "libbrute.so")
_brute = None


def load_golden(name: str):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def densify(F, C, K, rowptr, colidx, values):
    """CSR -> dense (F, C, K, K), written here from PAPER.md L391 (inverse of the flattening)."""
    w = np.zeros((F, C * K * K), np.float32)
    for f in range(F):
        for j in range(int(rowptr[f]), int(rowptr[f + 1])):
            w[f, int(colidx[j])] = values[j]
    return w.reshape(F, C, K, K)


def csr_from_dense(w):
    """Dense (F, C, K, K) -> CSR (rowptr, colidx, values), exact zeros dropped."""
    F = w.shape[0]
    flat = w.reshape(F, -1)
    rowptr = [0]
    cols, vals = [], []
    for f in range(F):
        nz = np.nonzero(flat[f])[0]
        cols.extend(nz.tolist())
        vals.extend(flat[f, nz].tolist())
        rowptr.append(len(cols))
    return (np.array(rowptr, np.int32), np.array(cols, np.int32), np.array(vals, np.float32))


def brute_dense_f32(x, wdense, bias, stride, pad):
    global _brute
    if _brute is None:
        if not os.path.exists(_BRUTE_LIB) or os.path.getmtime(_BRUTE_LIB) < os.path.getmtime(_BRUTE_SRC):
            tmp = _BRUTE_LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-ffp-contract=off",
                                   _BRUTE_SRC, "-o", tmp, "-lm"])
            os.replace(tmp, _BRUTE_LIB)
        _brute = ctypes.CDLL(_BRUTE_LIB)
        f32p = ctypes.POINTER(ctypes.c_float)
        _brute.brute_dense_conv_f32.argtypes = [ctypes.c_int] * 8 + [f32p] * 4
    x = np.ascontiguousarray(x, np.float32)
    wdense = np.ascontiguousarray(wdense, np.float32)
    N, C, H, W = x.shape
    F, _, K, _ = wdense.shape
    Ho = (H + 2 * pad - K) // stride + 1
    Wo = (W + 2 * pad - K) // stride + 1
    y = np.empty((N, F, Ho, Wo), np.float32)
    b = None if bias is None else np.ascontiguousarray(bias, np.float32)
    p = lambda a: None if a is None else a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
    st = _brute.brute_dense_conv_f32(N, C, H, W, F, K, stride, pad, p(wdense), p(b), p(x), p(y))
    assert st == 0
    return y


def bits(a):
    """float32 array -> uint32 bit patterns (for bitwise comparisons)."""
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def allclose_contract(got, ref, rtol=1e-5, atol=1e-4):
    """north_star tolerance: |g - o| <= atol + rtol*|o| (BASELINE.json)."""
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    err = np.abs(got - ref)
    bound = atol + rtol * np.abs(ref)
    return bool(np.all(err <= bound)), float(np.max(err / bound)) if err.size else 0.0
