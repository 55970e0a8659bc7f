"""cProfile of steady-state e2e segments (bench.py config B / D): where
the host-side Python of set-state / run / snapshot goes."""
import cProfile
import pstats
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig  # noqa: E402
from paper_1911_10274_b200 import io as sio  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0)
k = args.steps
ctl = SimController(st, env, cfg)
for rep in range(6):
    ctl.start(k * 1e-4)
    ctl.wait_for_event()
    snap = ctl.snapshot()
ids = snap.ids.copy()
pos_in = bench._native_pinned_copy(snap.positions)
vel_in = bench._native_pinned_copy(snap.velocities)
del snap
prof = cProfile.Profile()
for rep in range(40):
    prof.enable()
    sio.apply_snapshot(st, ids, pos_in, vel_in)
    ctl.start(k * 1e-4)
    ctl.wait_for_event()
    snap = ctl.snapshot()
    prof.disable()
    del snap
ctl.stop()
s = pstats.Stats(prof)
s.sort_stats("tottime").print_stats(30)
