"""Thin binding of the sparse multilayer LSTM C-ABI (include/spconv_lstm.h; SURVEY.md
§8(f) NEXT-4) — argument marshalling only; every step runs in libspconv.so's kernels."""
from __future__ import annotations

import ctypes

import numpy as np

from .spconv import SpconvError, _check, _ptr, _stream_handle, load_library

WAVEFRONT, SEQUENTIAL = 0, 1
EXPORTS = ("spconv_lstm_create", "spconv_lstm_forward", "spconv_lstm_launches", "spconv_lstm_destroy")


def _lib():
    lib = load_library()
    if not getattr(lib, "_lstm_bound", False):
        vp, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        lib.spconv_lstm_create.argtypes = [ctypes.POINTER(vp), I, I, I, vp, vp, vp, vp, vp, I]
        lib.spconv_lstm_forward.argtypes = [vp, I, I, vp, vp, I, vp]
        lib.spconv_lstm_launches.argtypes = [vp, I, I]
        lib.spconv_lstm_destroy.argtypes = [vp]
        for n in EXPORTS:
            getattr(lib, n).restype = I
        lib._lstm_bound = True
    return lib


class SparseLSTM:
    """Multilayer LSTM whose fused gate matrices [W_l | U_l] (4H x (D_l + H), gate rows
    i, f, g, o) are CSR; ``layers`` = [(rowptr, colidx, values, bias), ...]."""

    def __init__(self, D: int, H: int, layers, device: int = 0):
        self.L, self.D, self.H = len(layers), D, H
        rp = np.ascontiguousarray(np.concatenate([np.asarray(l[0], np.int32) for l in layers]))
        off = np.zeros(self.L + 1, np.int64)
        off[1:] = np.cumsum([len(l[1]) for l in layers])
        ci = np.ascontiguousarray(np.concatenate([np.asarray(l[1], np.int32) for l in layers]))
        vv = np.ascontiguousarray(np.concatenate([np.asarray(l[2], np.float32) for l in layers]))
        bias = [l[3] for l in layers]
        bb = None if all(b is None for b in bias) else np.ascontiguousarray(np.concatenate(
            [np.zeros(4 * H, np.float32) if b is None else np.asarray(b, np.float32) for b in bias]))
        self._keep = (rp, off, ci, vv, bb)
        h = ctypes.c_void_p()
        _check(_lib().spconv_lstm_create(ctypes.byref(h), self.L, D, H, _ptr(rp), _ptr(off), _ptr(ci),
                                         _ptr(vv), _ptr(bb), device), "spconv_lstm_create")
        self.plan = h

    def forward(self, x, schedule: int = WAVEFRONT, out=None, stream=None):
        """x: float32 CUDA tensor [T, B, D] -> the last layer's h [T, B, H]."""
        import torch
        if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 3 and
                x.shape[2] == self.D):
            raise ValueError("x must be a contiguous float32 CUDA tensor [T, B, D]")
        T, B, _ = x.shape
        if out is None:
            out = torch.empty((T, B, self.H), dtype=torch.float32, device=x.device)
        _check(_lib().spconv_lstm_forward(self.plan, T, B, x.data_ptr(), out.data_ptr(), schedule,
                                          _stream_handle(stream)), "spconv_lstm_forward")
        return out

    __call__ = forward

    def launches(self, T: int, schedule: int = WAVEFRONT) -> int:
        n = _lib().spconv_lstm_launches(self.plan, T, schedule)
        if n < 0:
            raise SpconvError(n, "spconv_lstm_launches")
        return n

    def close(self):
        if self.plan:
            _lib().spconv_lstm_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
