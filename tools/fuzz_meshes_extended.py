"""Extended campaign of tests/test_gpu_fuzz.py: random meshes (banded,
long-range, many components; random materials, actuation, yield, fixed
masses, contacts) stepped on the device against the oracle -- fp64 bit for
bit, fp32 / mixed within the tests' tolerance -- for many seeds."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import test_gpu_fuzz as t  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
fails = 0
cases = 0
t0 = time.time()
for shape in ("banded", "longrange", "components"):
    for seed in range(n):
        for prec in ("fp64", "fp32", "mixed"):
            cases += 1
            try:
                if prec == "fp64":
                    t.test_fuzz_fp64_bit_exact(seed, shape)
                else:
                    t.test_fuzz_tolerance_modes(seed, shape, prec)
                status = "ok"
            except Exception as exc:  # noqa: BLE001
                fails += 1
                status = f"FAIL {type(exc).__name__}: {str(exc)[:200]}"
            print(f"{shape} seed {seed} {prec}: {status}", flush=True)
print(f"{cases} cases, {fails} failures, {time.time() - t0:.1f} s")
