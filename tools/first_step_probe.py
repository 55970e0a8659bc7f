"""Device time of the first step of an sl_step call vs the host gap before
the call (SL_FIRST_STEP_MS=1 prints the split): is the first step's extra
cost idle wake-up or per-call work?"""
import os
import sys
import time

os.environ["SL_FIRST_STEP_MS"] = "1"
sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, engine  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision="fp32", device=0)
mir = engine.mirror_for(st, cfg)
mir.push(st, env)
ctx = mir.ctx
cnt = np.zeros(3, np.int64)
t = 0.0
for gap in (0.0, 0.0, 0.0001, 0.001, 0.01, 0.1, 0.0, 0.0):
    times = t + np.arange(20) * 1e-4
    t += 20e-4
    if gap:
        end = time.perf_counter() + gap
        while time.perf_counter() < end:
            pass
    sys.stderr.write(f"gap {gap * 1e3:.1f} ms: ")
    sys.stderr.flush()
    ctx.step(times, 1e-4, 0, cnt)
