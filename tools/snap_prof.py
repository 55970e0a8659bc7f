"""Snapshot latency right after a run ends vs after the controller thread
has settled (bench.py's e2e region ends with a snapshot)."""
import sys
import time
sys.path.insert(0, ".")
sys.argv = [sys.argv[0]] + sys.argv[1:]
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402
args = bench.parse()
st, env, *_ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision="fp32", device=0)
ctl = SimController(st, env, cfg)
for settle in (0.0, 0.05, 0.0, 0.05):
    ctl.start(args.steps * 1e-4)
    ctl.wait_for_event(timeout=60)
    if settle:
        time.sleep(settle)
    t = time.perf_counter()
    ctl.snapshot()
    print(f"settle {settle}: snapshot {1e3 * (time.perf_counter() - t):.2f} ms")
ctl.stop()
