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
    assert C.sizeof(_native.SlStats) == 8 * 8 + 4 * 4 + 3 * 8 + 2 * 4 + 8


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


def test_fp64_kernels_only_in_the_strict_unit(tmp_path):
    """Every fp64 (P = 0) kernel instantiation lives in the -fmad=false
    unit only.  A copy compiled with FMA contraction in another unit (the
    fp32 unit once instantiated k_win_tma<fp64> through an inline launcher)
    can be the one a launch binds to once that module is loaded, which
    broke fp64 bit-exactness after an fp32 context had run."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    subprocess.run([tool, "-xelf", "all", _native.LIB_PATH], cwd=tmp_path,
                   check=True, capture_output=True)
    cubins = sorted(p for p in os.listdir(tmp_path) if p.endswith(".cubin"))
    assert any("sl_kernels_fp64" in p for p in cubins)
    for p in cubins:
        out = subprocess.run([tool, "-symbols", str(tmp_path / p)],
                             check=True, capture_output=True, text=True)
        fp64 = [ln.split()[-1] for ln in out.stdout.splitlines()
                if "FUNC" in ln and re.search(r"_ZN2sl\d+k_\w+ILi0E",
                                              ln.split()[-1])
                and "$" not in ln.split()[-1]]
        if "sl_kernels_fp64" in p:
            assert any("k_win_tma" in s for s in fp64)
        else:
            assert fp64 == [], (p, fp64)
