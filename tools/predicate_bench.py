"""Condition-breakpoint cost on config B (100^3, fp32): a predicate checked
every N steps over K steps, synchronous checks (SL_NO_SPECULATE=1) against
speculative ones (the batch after a check runs while the host evaluates the
predicate on a checkpoint)."""
import os
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig  # noqa: E402
from paper_1911_10274_b200.control import Breakpoint, SimController  # noqa

st, env = bench.build_workload(100)
cfg = StepConfig(dt=1e-4, precision="fp32")
ctl = SimController(st, env, cfg)
ctl.start(20 * 1e-4)
ctl.wait_for_event()
for every in (10, 50):
    for spec in (False, True):
        if spec:
            os.environ.pop("SL_NO_SPECULATE", None)
        else:
            os.environ["SL_NO_SPECULATE"] = "1"
        ctl.set_breakpoint(Breakpoint.on_condition(
            lambda v: float(v.positions[:, 2].min()) < -1.0, every=every))
        k = 400
        w0 = time.perf_counter()
        ctl.start(k * 1e-4)
        rep = ctl.wait_for_event()
        wall = time.perf_counter() - w0
        print(f"every {every:3d} {'speculative' if spec else 'synchronous'}:"
              f" {1e3 * wall / k:.3f} ms/step over {k} steps "
              f"(reason {rep.reason})")
        ctl._conditions.clear()
ctl.stop()
