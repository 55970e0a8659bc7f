import sys, time
sys.path.insert(0, ".")
import bench
from paper_1911_10274_b200 import StepConfig, engine
from paper_1911_10274_b200.control import SimController
args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision="fp32", device=0)
ctl = SimController(st, env, cfg)
mir = engine.mirror_for(st, cfg)
orig = mir.ctx.step
sizes = []
def step(times, *a, **k):
    sizes.append(len(times))
    return orig(times, *a, **k)
mir.ctx.step = step
for rep in range(4):
    sizes.clear()
    ctl.start(20 * 1e-4)
    ctl.wait_for_event()
    print("rep", rep, sizes, ctl._sec_per_step)
    ctl.snapshot()
ctl.stop()
