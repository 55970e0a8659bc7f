"""The C-ABI library on CPU: it loads, exports every symbol
include/softlat_cuda.h declares, and fails cleanly (status codes, no crash)
when no device is present.  No compute calls here."""
import ctypes as C
import os
import re

import pytest

from paper_1911_10274_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "softlat_cuda.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sl_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_binding():
    assert declared_symbols() == sorted(_native.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # nothing but the ABI is exported (version script, _build.py)
    out = os.popen(f"nm -D --defined-only {_native.LIB_PATH}").read()
    exported = {ln.split()[-1] for ln in out.splitlines()
                if " T " in ln}
    assert exported == set(declared_symbols())


def test_abi_version_and_constants():
    lib = _native.load_library()
    assert lib.sl_abi_version() == 1
    hdr = open(HEADER).read()
    consts = dict(re.findall(r"#define (SL_\w+) (\d+)", hdr))
    assert int(consts["SL_OK"]) == _native.SL_OK
    assert int(consts["SL_ENUMERIC"]) == _native.SL_ENUMERIC
    assert int(consts["SL_ACC_GATHER"]) == _native.ACC_GATHER
    assert int(consts["SL_ACC_ATOMIC"]) == _native.ACC_ATOMIC
    assert int(consts["SL_ACC_AUTO"]) == _native.ACC_AUTO
    for name, code in _native.PRECISIONS.items():
        key = {"fp64": "SL_PREC_FP64", "fp32": "SL_PREC_FP32",
               "mixed": "SL_PREC_MIXED"}[name]
        assert int(consts[key]) == code
    assert C.sizeof(_native.SlStats) == 8 * 8 + 4 * 4 + 3 * 8


@pytest.mark.skipif(_native.device_count() > 0, reason="GPU present")
def test_no_device_fails_loudly_not_silently():
    """Without a GPU there is no fallback: context creation reports a CUDA
    error through the status code and sl_last_error."""
    lib = _native.load_library()
    h = C.c_void_p()
    rc = lib.sl_create(0, 1, C.byref(h))
    assert rc == _native.SL_ECUDA
    assert not h.value
    msg = lib.sl_last_error(None)
    assert msg and len(msg) > 0
    with pytest.raises(Exception):
        _native.Context(0, "fp32")


def test_bad_arguments_rejected_before_any_device_work():
    lib = _native.load_library()
    assert lib.sl_create(0, 7, None) == _native.SL_EINVAL
    h = C.c_void_p()
    assert lib.sl_create(0, 9, C.byref(h)) == _native.SL_EINVAL
    assert lib.sl_step(None, 1, None, 1e-4, 0, None, None, None) == \
        _native.SL_EINVAL
