"""Thin Python binding of libspconv.so (include/spconv.h) — argument marshalling only.

Every function here forwards to the C-ABI entry point of the same name; every
step of the hot path runs in the library's CUDA kernels.  PyTorch is used only
for device memory and streams.  If the library is missing or no CUDA device is
present the calls raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
# SPCONV_LIB: load another build of the same ABI (A/B timing of kernel changes)
LIB_PATH = os.environ.get("SPCONV_LIB") or os.path.join(_PKG, "libspconv.so")

SPCONV_OK = 0
STATUS = {0: "OK", -1: "NULLPTR", -2: "SHAPE", -3: "CSR", -4: "UNSUPPORTED", -5: "ALIGN",
          -6: "DEVICE", -7: "CUDA", -8: "OOM", -9: "ALIAS", -10: "INTERNAL"}
KERNEL_AUTO, KERNEL_GENERIC, KERNEL_TILED, KERNEL_PIPE, KERNEL_DENSE = 0, 1, 2, 3, 4
KERNELS = {"auto": KERNEL_AUTO, "generic": KERNEL_GENERIC, "tiled": KERNEL_TILED, "pipe": KERNEL_PIPE,
           "dense": KERNEL_DENSE}

# Every symbol include/spconv.h declares (checked by tests/test_abi.py).
EXPORTS = ("spconv_create", "spconv_create_ex", "spconv_forward", "spconv_fused_relu_maxpool",
           "spconv_forward_host", "spconv_destroy", "spconv_output_dims", "spconv_plan_info",
           "spconv_status_string", "spconv_abi_version", "spconv_debug_decoded",
           "spconv_last_cuda_error", "spconv_forward_ex", "spconv_resize_bilinear",
           "spconv_resize_fused_relu_maxpool", "spconv_launch_info", "spconv_debug_sk_split")


class SpconvError(RuntimeError):
    def __init__(self, status: int, what: str):
        self.status = status
        msg = f"{what}: {STATUS.get(status, status)} ({status_string(status)})"
        if status == -7 and _lib is not None:
            msg += f": {_lib.spconv_last_cuda_error().decode()}"
        super().__init__(msg)


class Options(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("rows_per_group", ctypes.c_int),
                ("reserved", ctypes.c_int * 6)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("C", ctypes.c_int), ("H", ctypes.c_int), ("W", ctypes.c_int), ("F", ctypes.c_int),
                ("K", ctypes.c_int), ("stride", ctypes.c_int), ("pad", ctypes.c_int),
                ("Ho", ctypes.c_int), ("Wo", ctypes.c_int), ("nnz", ctypes.c_int64),
                ("device", ctypes.c_int), ("kernel", ctypes.c_int), ("rows_per_group", ctypes.c_int),
                ("num_groups", ctypes.c_int), ("device_bytes", ctypes.c_int64),
                ("launches_per_call", ctypes.c_int)]


class LaunchInfo(ctypes.Structure):
    _fields_ = [("kernel", ctypes.c_int), ("rows_per_group", ctypes.c_int), ("grid", ctypes.c_int),
                ("stream_k", ctypes.c_int), ("units", ctypes.c_int64), ("band", ctypes.c_int),
                ("staging", ctypes.c_int), ("channels_per_stage", ctypes.c_int), ("stages", ctypes.c_int),
                ("launches", ctypes.c_int), ("tile_rows", ctypes.c_int), ("sk_split", ctypes.c_int),
                ("reserved", ctypes.c_int * 5)]


_lib = None


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libspconv.so (raises if it was not built: run __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} not found — build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    vp, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    lib.spconv_create.argtypes = [ctypes.POINTER(vp), I, I, I, I, I, I, I, vp, vp, vp, L, vp, I]
    lib.spconv_create_ex.argtypes = lib.spconv_create.argtypes + [ctypes.POINTER(Options)]
    lib.spconv_forward.argtypes = [vp, I, vp, vp, vp]
    lib.spconv_fused_relu_maxpool.argtypes = [vp, I, vp, vp, vp, vp]
    lib.spconv_forward_ex.argtypes = [vp, I, vp, vp, vp, I, vp]
    lib.spconv_resize_bilinear.argtypes = [I, I, vp, I, I, vp, I, I, vp]
    lib.spconv_resize_fused_relu_maxpool.argtypes = [vp, I, vp, I, I, vp, vp, vp]
    lib.spconv_forward_host.argtypes = [vp, I, vp, vp, I, vp]
    lib.spconv_destroy.argtypes = [vp]
    lib.spconv_output_dims.argtypes = [vp, I, I, ctypes.POINTER(ctypes.c_int64)]
    lib.spconv_plan_info.argtypes = [vp, ctypes.POINTER(PlanInfo)]
    if hasattr(lib, "spconv_launch_info") or path == os.path.join(_PKG, "libspconv.so"):
        # (A/B tooling may load an older build through SPCONV_LIB that predates it)
        lib.spconv_launch_info.argtypes = [vp, I, I, vp, ctypes.POINTER(LaunchInfo)]
    lib.spconv_status_string.argtypes = [I]
    lib.spconv_status_string.restype = ctypes.c_char_p
    lib.spconv_abi_version.argtypes = []
    lib.spconv_last_cuda_error.argtypes = []
    lib.spconv_last_cuda_error.restype = ctypes.c_char_p
    lib.spconv_debug_decoded.argtypes = [vp, vp, vp, vp]
    if hasattr(lib, "spconv_debug_sk_split"):
        lib.spconv_debug_sk_split.argtypes = [vp, I, I, I, I, I, L, I, I, vp, vp]
    for name in EXPORTS:
        if name not in ("spconv_status_string", "spconv_last_cuda_error") and hasattr(lib, name):
            getattr(lib, name).restype = I
    _lib = lib
    return lib


def status_string(status: int) -> str:
    try:
        return load_library().spconv_status_string(status).decode()
    except ImportError:
        return STATUS.get(status, "unknown")


def _check(status: int, what: str) -> None:
    if status != SPCONV_OK:
        raise SpconvError(status, what)


def _ptr(a) -> int | None:
    """Address of a numpy array or torch tensor (host or device), None for None."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch.Tensor


def _as_c(a, dtype):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=dtype)
    import torch
    tdt = {np.int32: torch.int32, np.float32: torch.float32}[dtype]
    return a.to(tdt).contiguous()


def _stream_handle(stream) -> int | None:
    if stream is None:
        import torch
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


# ---------------------------------------------------------------- C-ABI names
def spconv_create(C, H, W, F, K, stride, pad, rowptr, colidx, values, bias=None, device=0,
                  kernel: str = "auto", rows_per_group: int = 0) -> int:
    """Returns an opaque plan handle (int).  CSR/bias may be numpy arrays or torch tensors
    (host or device); they are deep-copied."""
    lib = load_library()
    rowptr = _as_c(rowptr, np.int32)
    colidx = _as_c(colidx, np.int32)
    values = _as_c(values, np.float32)
    bias = _as_c(bias, np.float32)
    nnz = int(colidx.shape[0])
    h = ctypes.c_void_p()
    opts = Options(KERNELS[kernel], rows_per_group)
    st = lib.spconv_create_ex(ctypes.byref(h), C, H, W, F, K, stride, pad, _ptr(rowptr), _ptr(colidx),
                              _ptr(values), nnz, _ptr(bias), device, ctypes.byref(opts))
    _check(st, "spconv_create")
    return h.value


def spconv_forward(plan, N, x_ptr, y_ptr, stream=None) -> None:
    _check(load_library().spconv_forward(plan, N, x_ptr, y_ptr, _stream_handle(stream)), "spconv_forward")


EPI_RELU, EPI_RESIDUAL = 1, 2


def spconv_resize_bilinear(N, C, x_ptr, Hin, Win, y_ptr, Hout, Wout, stream=None) -> None:
    _check(load_library().spconv_resize_bilinear(N, C, x_ptr, Hin, Win, y_ptr, Hout, Wout,
                                                 _stream_handle(stream)), "spconv_resize_bilinear")


def spconv_resize_fused_relu_maxpool(plan, N, x_ptr, Hin, Win, y_ptr, argmax_ptr=None, stream=None) -> None:
    _check(load_library().spconv_resize_fused_relu_maxpool(plan, N, x_ptr, Hin, Win, y_ptr, argmax_ptr,
                                                           _stream_handle(stream)),
           "spconv_resize_fused_relu_maxpool")


def spconv_forward_ex(plan, N, x_ptr, residual_ptr, y_ptr, flags, stream=None) -> None:
    _check(load_library().spconv_forward_ex(plan, N, x_ptr, residual_ptr, y_ptr, flags,
                                            _stream_handle(stream)), "spconv_forward_ex")


def spconv_fused_relu_maxpool(plan, N, x_ptr, y_ptr, argmax_ptr=None, stream=None) -> None:
    _check(load_library().spconv_fused_relu_maxpool(plan, N, x_ptr, y_ptr, argmax_ptr,
                                                    _stream_handle(stream)), "spconv_fused_relu_maxpool")


def spconv_forward_host(plan, N, x_host: np.ndarray, y_host: np.ndarray, fused=False, argmax_host=None):
    _check(load_library().spconv_forward_host(plan, N, _ptr(x_host), _ptr(y_host), int(bool(fused)),
                                              _ptr(argmax_host)), "spconv_forward_host")


def spconv_destroy(plan) -> None:
    if plan:
        load_library().spconv_destroy(plan)


def spconv_output_dims(plan, N, fused=False):
    dims = (ctypes.c_int64 * 4)()
    _check(load_library().spconv_output_dims(plan, N, int(bool(fused)), dims), "spconv_output_dims")
    return tuple(int(d) for d in dims)


def spconv_plan_info(plan) -> dict:
    info = PlanInfo()
    _check(load_library().spconv_plan_info(plan, ctypes.byref(info)), "spconv_plan_info")
    return {f: getattr(info, f) for f, _ in PlanInfo._fields_}


def spconv_launch_info(plan, N, fused=False, x_ptr=None) -> dict:
    """The launch schedule a forward of N images would use (stream-K, grid, units, ...)."""
    info = LaunchInfo()
    _check(load_library().spconv_launch_info(plan, N, int(bool(fused)), x_ptr, ctypes.byref(info)),
           "spconv_launch_info")
    return {f: getattr(info, f) for f, _ in LaunchInfo._fields_ if f != "reserved"}


def spconv_debug_sk_split(cost, C, gpc, ngs, num_groups, cc, units, grid, fused=False):
    """Test-only host call: the per-warp stream-K split table (unit[grid+1], ch[grid+1, gpc])
    for a float32 cost array [ngs, gpc, C]; raises SpconvError if no valid split exists."""
    cost = np.ascontiguousarray(cost, dtype=np.float32)
    assert cost.shape == (ngs, gpc, C)
    unit = np.zeros(grid + 1, np.int32)
    ch = np.zeros((grid + 1, gpc), np.uint16)
    _check(load_library().spconv_debug_sk_split(_ptr(cost), C, gpc, ngs, num_groups, cc, units, grid,
                                                int(bool(fused)), _ptr(unit), _ptr(ch)), "spconv_debug_sk_split")
    return unit, ch


def spconv_debug_decoded(plan, nnz):
    c, dy, dx = (np.empty(nnz, np.int32) for _ in range(3))
    _check(load_library().spconv_debug_decoded(plan, _ptr(c), _ptr(dy), _ptr(dx)), "spconv_debug_decoded")
    return c, dy, dx


# ---------------------------------------------------------------- convenience object
class SparseConv2d:
    """A CSR sparse conv layer bound to one CUDA device (a plan + torch-tensor calls).

    Parameters follow PAPER.md's problem statement: C, H, W (input), F output
    channels, K x K filters, stride, pad, CSR rowptr/colidx/values over the
    flattened (F, C*K*K) filter matrix, optional bias.
    """

    def __init__(self, C, H, W, F, K, stride, pad, rowptr, colidx, values, bias=None, device=0,
                 kernel="auto", rows_per_group=0):
        self.C, self.H, self.W, self.F, self.K, self.stride, self.pad = C, H, W, F, K, stride, pad
        self.device = device
        self.nnz = int(len(colidx))
        self.plan = spconv_create(C, H, W, F, K, stride, pad, rowptr, colidx, values, bias, device,
                                  kernel, rows_per_group)
        self.info = spconv_plan_info(self.plan)
        self.Ho, self.Wo = self.info["Ho"], self.info["Wo"]

    def close(self):
        if self.plan:
            spconv_destroy(self.plan)
            self.plan = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def output_shape(self, N, fused=False):
        return spconv_output_dims(self.plan, N, fused)

    def _check_x(self, x):
        import torch
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32):
            raise TypeError("x must be a CUDA float32 tensor (no CPU fallback)")
        if x.dim() != 4 or tuple(x.shape[1:]) != (self.C, self.H, self.W):
            raise ValueError(f"x shape {tuple(x.shape)} != (N, {self.C}, {self.H}, {self.W})")
        return x.contiguous()

    def forward(self, x, out=None, stream=None):
        import torch
        x = self._check_x(x)
        N = x.shape[0]
        if out is None:
            out = torch.empty(self.output_shape(N), dtype=torch.float32, device=x.device)
        spconv_forward(self.plan, N, x.data_ptr(), out.data_ptr(), stream)
        return out

    __call__ = forward

    def forward_ex(self, x, relu=False, residual=None, out=None, stream=None):
        """y = [ReLU]((conv(x) + bias) [+ residual]) (spconv_forward_ex)."""
        import torch
        x = self._check_x(x)
        N = x.shape[0]
        if out is None:
            out = torch.empty(self.output_shape(N), dtype=torch.float32, device=x.device)
        flags = (EPI_RELU if relu else 0) | (EPI_RESIDUAL if residual is not None else 0)
        if residual is not None:
            if tuple(residual.shape) != tuple(out.shape) or residual.dtype != torch.float32 or \
                    not residual.is_contiguous():
                raise ValueError("residual must be a contiguous float32 tensor of the output shape")
        spconv_forward_ex(self.plan, N, x.data_ptr(), None if residual is None else residual.data_ptr(),
                          out.data_ptr(), flags, stream)
        return out

    def fused_relu_maxpool(self, x, out=None, argmax=None, with_argmax=True, stream=None):
        import torch
        x = self._check_x(x)
        N = x.shape[0]
        shp = self.output_shape(N, fused=True)
        if out is None:
            out = torch.empty(shp, dtype=torch.float32, device=x.device)
        if argmax is None and with_argmax:
            argmax = torch.empty(shp, dtype=torch.int32, device=x.device)
        spconv_fused_relu_maxpool(self.plan, N, x.data_ptr(), out.data_ptr(),
                                  None if argmax is None else argmax.data_ptr(), stream)
        return out, argmax

    def resize_fused_relu_maxpool(self, x, with_argmax=True, stream=None):
        """maxpool2x2(ReLU(conv(resize(x)) + bias)), x of any spatial size (NEXT-2)."""
        import torch
        if not (x.is_cuda and x.dtype == torch.float32 and x.is_contiguous() and x.dim() == 4 and
                x.shape[1] == self.C):
            raise ValueError("x must be a contiguous float32 CUDA tensor [N, C, Hin, Win]")
        N, _, Hin, Win = x.shape
        shp = self.output_shape(N, fused=True)
        out = torch.empty(shp, dtype=torch.float32, device=x.device)
        am = torch.empty(shp, dtype=torch.int32, device=x.device) if with_argmax else None
        spconv_resize_fused_relu_maxpool(self.plan, N, x.data_ptr(), Hin, Win, out.data_ptr(),
                                         None if am is None else am.data_ptr(), stream)
        return out, am

    def forward_host(self, x: np.ndarray, fused=False, with_argmax=True):
        x = np.ascontiguousarray(x, np.float32)
        N = x.shape[0]
        y = np.empty(self.output_shape(N, fused), np.float32)
        am = np.empty(y.shape, np.int32) if (fused and with_argmax) else None
        spconv_forward_host(self.plan, N, x, y, fused, am)
        return (y, am) if fused else y

    def launch_info(self, N, fused=False, x=None):
        return spconv_launch_info(self.plan, N, fused, None if x is None else x.data_ptr())

    def debug_decoded(self):
        return spconv_debug_decoded(self.plan, self.nnz)
