"""In-tree build of libsoftlat_cuda.so (sm_100a) with nvcc.

The library is the product's compute path; it is built next to this file so
the .so travels with the repo snapshot to the GPU box.  Translation units:

* csrc/sl_kernels_fp64.cu -- fp64 parity kernels, ``-fmad=false`` so every
  multiply and add rounds separately, as the reference's numba kernels do
  (kernels.py is compiled without fastmath; SURVEY.md 7 hard part 2).
* csrc/sl_kernels_fp32.cu -- fp32 / mixed kernels (FMA allowed).
* csrc/sl_api.cu          -- context, layout build (CUB), C ABI.
* csrc/sl_host.cpp        -- host-side snapshot formatting, lattice generation,
  parallel fills (threads; no FMA contraction: bit-exact with numpy).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB_NAME = "libsoftlat_cuda.so"
LIB_PATH = os.path.join(HERE, LIB_NAME)
OBJ_DIR = os.path.join(HERE, "build")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
          "-I", INCLUDE, "-I", CSRC]
UNITS = {
    "sl_kernels_fp64.cu": ["-fmad=false"],
    # tolerance modes: flush denormals (keeps MUFU.RSQ free of the
    # denormal-rescaling sequence); IEEE divide/sqrt are not used there
    "sl_kernels_fp32.cu": ["-ftz=true"],
    "sl_api.cu": [],
    "sl_host.cpp": ["-Xcompiler", "-ffp-contract=off"],  # host only
}


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc",
                 shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; cannot build libsoftlat_cuda.so")


def _deps() -> list[str]:
    out = [os.path.join(INCLUDE, "softlat_cuda.h"), __file__]
    for f in os.listdir(CSRC):
        out.append(os.path.join(CSRC, f))
    return out


def up_to_date() -> bool:
    if not os.path.exists(LIB_PATH):
        return False
    if any(k.startswith("SL_NVCC_") for k in os.environ):
        return False
    t = os.path.getmtime(LIB_PATH)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB_PATH
    os.makedirs(OBJ_DIR, exist_ok=True)
    cc = nvcc()
    objs = []
    procs = []
    for unit, extra in UNITS.items():
        obj = os.path.join(OBJ_DIR, os.path.splitext(unit)[0] + ".o")
        # tuning sweeps: extra flags for one unit, e.g.
        # SL_NVCC_sl_kernels_fp64="-DWIN_XU=3 -DSL_WIN64_T=11"
        tune = os.environ.get("SL_NVCC_" + os.path.splitext(unit)[0])
        if tune:
            extra = extra + tune.split()
        cmd = [cc, *ARCH, *COMMON, *extra, "-c", os.path.join(CSRC, unit),
               "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT,
                                            text=True)))
        objs.append(obj)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{out}")
        if verbose and out:
            print(out, file=sys.stderr)
    vs = os.path.join(OBJ_DIR, "exports.map")
    with open(vs, "w") as fh:
        fh.write("{ global: sl_*; local: *; };\n")
    tmp = LIB_PATH + ".tmp"
    cmd = [cc, *ARCH, "-shared", "-o", tmp, *objs,
           "-Xlinker", f"--version-script={vs}"]
    subprocess.run(cmd, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
