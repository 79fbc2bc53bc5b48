"""CPU oracle for the CSR sparse direct convolution (arXiv 2005.04091).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2005_04091_b200``) never imports it and
shares no code with it.

The arithmetic lives in ``spconv_oracle.c`` (plain C, each function citing the
PAPER.md passage it follows); this file only builds it with gcc and marshals
numpy arrays.  Pins: ``tests/test_oracle_pins.py``.  Parity pinned: decode,
conv (f32-ordered and f64), fused ReLU+maxpool+argmax, point queries.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "spconv_oracle.c")
_SRC_LSTM = os.path.join(_HERE, "lstm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
# No -ffast-math, no FMA contraction of the plain expressions; fmaf() is the
# only fused operation (reading G7 in DESIGN.md).
CFLAGS = ["-O2", "-fPIC", "-shared", "-pthread", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]

# ORACLE_SANITIZE=1: load a build instrumented with AddressSanitizer + UBSan (SURVEY.md
# §5: "the host oracle under -fsanitize=address,undefined"; tests/test_oracle_sanitized.py
# runs it in a subprocess with the ASan runtime preloaded)
SANITIZE = os.environ.get("ORACLE_SANITIZE") == "1"
if SANITIZE:
    _LIB = os.path.join(_HERE, "liboracle_san.so")
    CFLAGS = CFLAGS + ["-g", "-O1", "-fno-omit-frame-pointer", "-fsanitize=address,undefined",
                       "-fno-sanitize-recover=all"]

_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (checker only; not the product)."""
    srcs = [_SRC, _SRC_LSTM]
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in srcs):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, *srcs, "-o", tmp, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i32p = ctypes.POINTER(ctypes.c_int32)
        f32p = ctypes.POINTER(ctypes.c_float)
        f64p = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        I, L = ctypes.c_int, ctypes.c_int64
        shape = [I] * 8
        lib.oracle_check_csr.argtypes = [I, I, I, i32p, i32p, f32p, L]
        lib.oracle_decode.argtypes = [I, L, i32p, i32p, i32p, i32p]
        lib.oracle_decode.restype = None
        lib.oracle_conv_f32.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, f32p, I]
        lib.oracle_conv_f64.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, f64p, I]
        lib.oracle_fused_f32.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, f32p, i32p, I]
        lib.oracle_conv_points_f32.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, L, i64p, f32p]
        lib.oracle_conv_points_f64.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, L, i64p, f64p]
        lib.oracle_fused_points_f32.argtypes = shape + [i32p, i32p, f32p, f32p, f32p, L, i64p,
                                                         f32p, i32p]
        lib.oracle_epilogue_f32.argtypes = [f32p, f32p, L, I]
        lib.oracle_resize_bilinear_f32.argtypes = [I, I, I, I, I, I, f32p, f32p]
        lib.oracle_resize_bilinear_f32.restype = None
        lib.oracle_lstm_f64.argtypes = [I, I, I, I, I, i32p, i64p, i32p, f32p, f32p, f32p, f64p]
        lib.oracle_epilogue_f32.restype = None
        _lib = lib
    return _lib


def _p(a, ct):
    if a is None:
        return None
    return a.ctypes.data_as(ctypes.POINTER(ct))


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def out_dims(H, W, K, stride, pad):
    return (H + 2 * pad - K) // stride + 1, (W + 2 * pad - K) // stride + 1


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class OracleError(RuntimeError):
    pass


def _check(status):
    if status != 0:
        raise OracleError(f"oracle status {status}")


def check_csr(F, C, K, rowptr, colidx, values) -> int:
    lib = _load()
    rowptr, colidx, values = _c(rowptr, np.int32), _c(colidx, np.int32), _c(values, np.float32)
    return lib.oracle_check_csr(F, C, K, _p(rowptr, ctypes.c_int32), _p(colidx, ctypes.c_int32),
                                _p(values, ctypes.c_float), colidx.shape[0])


def decode(K, colidx):
    lib = _load()
    colidx = _c(colidx, np.int32)
    n = colidx.shape[0]
    c, ky, kx = (np.empty(n, np.int32) for _ in range(3))
    lib.oracle_decode(K, n, _p(colidx, ctypes.c_int32), _p(c, ctypes.c_int32),
                      _p(ky, ctypes.c_int32), _p(kx, ctypes.c_int32))
    return c, ky, kx


def _args(x, F, K, stride, pad, rowptr, colidx, values, bias):
    x = _c(x, np.float32)
    N, C, H, W = x.shape
    rowptr, colidx, values = _c(rowptr, np.int32), _c(colidx, np.int32), _c(values, np.float32)
    bias = _c(bias, np.float32)
    assert rowptr.shape[0] == F + 1
    keep = (x, rowptr, colidx, values, bias)
    args = [N, C, H, W, F, K, stride, pad, _p(rowptr, ctypes.c_int32), _p(colidx, ctypes.c_int32),
            _p(values, ctypes.c_float), _p(bias, ctypes.c_float), _p(x, ctypes.c_float)]
    return args, keep, (N, C, H, W)


def conv_f32(x, F, K, stride, pad, rowptr, colidx, values, bias=None, nthreads=None):
    """FP32-ordered conv (the parity contract, reading G7)."""
    lib = _load()
    args, keep, (N, C, H, W) = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    Ho, Wo = out_dims(H, W, K, stride, pad)
    y = np.empty((N, F, Ho, Wo), np.float32)
    _check(lib.oracle_conv_f32(*args, _p(y, ctypes.c_float), nthreads or default_threads()))
    return y


def conv_ex_f32(x, F, K, stride, pad, rowptr, colidx, values, bias=None, residual=None, relu=False,
                nthreads=None):
    """ReLU((conv + bias) + residual) in FP32, the block epilogue of NEXT-3 (R1)."""
    y = conv_f32(x, F, K, stride, pad, rowptr, colidx, values, bias, nthreads)
    flags = (1 if relu else 0) | (2 if residual is not None else 0)
    res = None
    if residual is not None:
        res = np.ascontiguousarray(residual, np.float32)
        if res.shape != y.shape:
            raise ValueError("residual shape mismatch")
    _load().oracle_epilogue_f32(_p(y, ctypes.c_float), None if res is None else _p(res, ctypes.c_float),
                                y.size, flags)
    return y


def resize_bilinear_f32(x, Hout, Wout):
    """Bilinear resize, half-pixel centres (reading R2), plain FP32."""
    x = np.ascontiguousarray(x, np.float32)
    N, C, Hin, Win = x.shape
    y = np.empty((N, C, Hout, Wout), np.float32)
    _load().oracle_resize_bilinear_f32(N, C, Hin, Win, Hout, Wout, _p(x, ctypes.c_float), _p(y, ctypes.c_float))
    return y


def conv_f64(x, F, K, stride, pad, rowptr, colidx, values, bias=None, nthreads=None):
    lib = _load()
    args, keep, (N, C, H, W) = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    Ho, Wo = out_dims(H, W, K, stride, pad)
    y = np.empty((N, F, Ho, Wo), np.float64)
    _check(lib.oracle_conv_f64(*args, _p(y, ctypes.c_double), nthreads or default_threads()))
    return y


def fused_f32(x, F, K, stride, pad, rowptr, colidx, values, bias=None, nthreads=None):
    """maxpool2x2(ReLU(conv + bias)) with first-max argmax."""
    lib = _load()
    args, keep, (N, C, H, W) = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    Ho, Wo = out_dims(H, W, K, stride, pad)
    y = np.empty((N, F, Ho // 2, Wo // 2), np.float32)
    am = np.empty((N, F, Ho // 2, Wo // 2), np.int32)
    _check(lib.oracle_fused_f32(*args, _p(y, ctypes.c_float), _p(am, ctypes.c_int32),
                                nthreads or default_threads()))
    return y, am


def conv_points_f32(x, F, K, stride, pad, rowptr, colidx, values, bias, pts):
    lib = _load()
    args, keep, _ = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    pts = _c(pts, np.int64).reshape(-1, 4)
    out = np.empty(pts.shape[0], np.float32)
    _check(lib.oracle_conv_points_f32(*args, pts.shape[0], _p(pts, ctypes.c_int64),
                                      _p(out, ctypes.c_float)))
    return out


def conv_points_f64(x, F, K, stride, pad, rowptr, colidx, values, bias, pts):
    lib = _load()
    args, keep, _ = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    pts = _c(pts, np.int64).reshape(-1, 4)
    out = np.empty(pts.shape[0], np.float64)
    _check(lib.oracle_conv_points_f64(*args, pts.shape[0], _p(pts, ctypes.c_int64),
                                      _p(out, ctypes.c_double)))
    return out


def fused_points_f32(x, F, K, stride, pad, rowptr, colidx, values, bias, pts):
    lib = _load()
    args, keep, _ = _args(x, F, K, stride, pad, rowptr, colidx, values, bias)
    pts = _c(pts, np.int64).reshape(-1, 4)
    out = np.empty(pts.shape[0], np.float32)
    am = np.empty(pts.shape[0], np.int32)
    _check(lib.oracle_fused_points_f32(*args, pts.shape[0], _p(pts, ctypes.c_int64),
                                       _p(out, ctypes.c_float), _p(am, ctypes.c_int32)))
    return out, am


def lstm_f64(x, layers, H):
    """Sparse multilayer LSTM (NEXT-4, reading R3), sequential, float64.

    x: float32 [T, B, D]; layers: list of (rowptr[4H+1], colidx, values, bias[4H]) CSR
    of the fused gate matrix [W | U] (4H x (D_l + H)), gate order i, f, g, o.
    Returns the last layer's h as float64 [T, B, H]."""
    x = np.ascontiguousarray(x, np.float32)
    T, B, D = x.shape
    L = len(layers)
    rp = np.concatenate([np.asarray(l[0], np.int32) for l in layers])
    nnz = [int(len(l[1])) for l in layers]
    off = np.zeros(L + 1, np.int64)
    off[1:] = np.cumsum(nnz)
    ci = np.ascontiguousarray(np.concatenate([np.asarray(l[1], np.int32) for l in layers]))
    vv = np.ascontiguousarray(np.concatenate([np.asarray(l[2], np.float32) for l in layers]))
    bb = np.ascontiguousarray(np.concatenate([np.asarray(l[3], np.float32) for l in layers]))
    h = np.empty((T, B, H), np.float64)
    st = _load().oracle_lstm_f64(L, D, H, T, B, _p(rp, ctypes.c_int32), _p(off, ctypes.c_int64),
                                 _p(ci, ctypes.c_int32), _p(vv, ctypes.c_float), _p(bb, ctypes.c_float),
                                 _p(x, ctypes.c_float), _p(h, ctypes.c_double))
    _check(st)
    return h
