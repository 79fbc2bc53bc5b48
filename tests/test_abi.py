"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/spconv.h declares, and refuses to run without a device (no CPU fallback)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "spconv.h")
HEADERS = sorted(os.path.join(ROOT, "include", h) for h in os.listdir(os.path.join(ROOT, "include"))
                 if h.endswith(".h"))


def _declared():
    names = set()
    for h in HEADERS:
        src = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        names |= set(re.findall(r"\b(spconv_[a-z_]+)\s*\(", src))
    return sorted(names)


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__.build_library()
    from paper_2005_04091_b200 import spconv
    return spconv.load_library()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("spconv_create", "spconv_forward", "spconv_fused_relu_maxpool", "spconv_destroy"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    from paper_2005_04091_b200 import spconv
    for name in _declared():
        assert hasattr(lib, name), name
    from paper_2005_04091_b200 import lstm
    assert set(_declared()) == set(spconv.EXPORTS) | set(lstm.EXPORTS)


def test_status_strings_and_version(lib):
    assert lib.spconv_abi_version() == 1
    for code in range(-9, 1):
        s = lib.spconv_status_string(code)
        assert s and s != b"unknown status"
    assert lib.spconv_status_string(-99) == b"unknown status"


def test_null_and_shape_errors_before_any_device_work(lib):
    h = ctypes.c_void_p()
    rp = np.zeros(3, np.int32)
    # NULL plan out-pointer / NULL rowptr
    assert lib.spconv_create(None, 1, 4, 4, 2, 3, 1, 1, rp.ctypes.data, None, None, 0, None, 0) == -1
    assert lib.spconv_create(ctypes.byref(h), 1, 4, 4, 2, 3, 1, 1, None, None, None, 0, None, 0) == -1
    # bad shapes
    assert lib.spconv_create(ctypes.byref(h), 0, 4, 4, 2, 3, 1, 1, rp.ctypes.data, None, None, 0, None, 0) == -2
    assert lib.spconv_create(ctypes.byref(h), 1, 1, 1, 2, 5, 1, 1, rp.ctypes.data, None, None, 0, None, 0) == -2
    # unsupported
    assert lib.spconv_create(ctypes.byref(h), 1, 16, 16, 2, 9, 1, 1, rp.ctypes.data, None, None, 0, None, 0) == -4
    # NULL plan handle on the run / query entry points
    assert lib.spconv_forward(None, 1, None, None, None) == -1
    assert lib.spconv_fused_relu_maxpool(None, 1, None, None, None, None) == -1
    assert lib.spconv_destroy(None) == 0


def test_no_cpu_fallback_without_a_device(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rp = np.array([0, 1], np.int32)
    ci = np.array([4], np.int32)
    v = np.array([1.0], np.float32)
    st = lib.spconv_create(ctypes.byref(h), 1, 4, 4, 1, 3, 1, 1, rp.ctypes.data, ci.ctypes.data,
                           v.ctypes.data, 1, None, 0)
    assert st in (-6, -7) and not h.value
    from paper_2005_04091_b200 import SparseConv2d, SpconvError
    with pytest.raises(SpconvError):
        SparseConv2d(1, 4, 4, 1, 3, 1, 1, rp, ci, v)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2005_04091_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".h", ".cpp", ".inc")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "spconv_oracle" not in text, f
