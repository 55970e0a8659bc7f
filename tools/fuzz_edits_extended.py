"""Extended campaign of tests/test_gpu_fuzz_edits.py: random edit sequences
(deletions, creations, re-wirings, retunes, mass deletions / creations,
constraints, loads) between runs against the oracle, many seeds, both
precisions; fp64 bit-exact.  Prints one line per case and a summary."""
import sys
import time

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
sys.path.insert(0, "oracle")
import test_gpu_fuzz_edits as t  # noqa: E402
from paper_1911_10274_b200 import _native  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
fails = 0
t0 = time.time()
for prec in ("fp64", "fp32"):
    for seed in range(n):
        try:
            t.test_random_edits_between_runs(seed, prec)
            status = "ok"
        except Exception as exc:  # noqa: BLE001
            fails += 1
            status = f"FAIL {type(exc).__name__}: {str(exc)[:200]}"
        print(f"{prec} seed {seed}: {status}", flush=True)
print(f"{2 * n} cases, {fails} failures, {time.time() - t0:.1f} s; "
      f"library {_native.LIB_PATH}")
