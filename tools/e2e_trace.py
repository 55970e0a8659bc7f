"""Per-call host timeline of steady-state e2e segments (bench.py config B):
every _native.Context method call with its wall time, in order, for the
last segments.  Tells where set-state / run / snapshot spend their time."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, _native  # noqa: E402
from paper_1911_10274_b200 import io as sio  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0)
k = args.steps
log = []
T0 = [0.0]


def wrap(name, f):
    def g(*a, **kw):
        t = time.perf_counter()
        try:
            return f(*a, **kw)
        finally:
            t2 = time.perf_counter()
            log.append((1e3 * (t - T0[0]), 1e3 * (t2 - t), name))
    return g


for name, f in list(vars(_native.Context).items()):
    if callable(f) and not name.startswith("_"):
        setattr(_native.Context, name, wrap(name, f))

ctl = SimController(st, env, cfg)
for rep in range(6):
    ctl.start(k * 1e-4)
    ctl.wait_for_event()
    snap = ctl.snapshot()
ids = snap.ids.copy()
pos_in = bench._native_pinned_copy(snap.positions)
vel_in = bench._native_pinned_copy(snap.velocities)
for rep in range(4):
    log.clear()
    T0[0] = t0 = time.perf_counter()
    sio.apply_snapshot(st, ids, pos_in, vel_in)
    t1 = time.perf_counter()
    ctl.start(k * 1e-4)
    ctl.wait_for_event()
    t2 = time.perf_counter()
    snap = ctl.snapshot()
    t3 = time.perf_counter()
    print(f"rep {rep}: set-state {1e3*(t1-t0):.2f} run {1e3*(t2-t1):.2f} "
          f"snapshot {1e3*(t3-t2):.2f} total {1e3*(t3-t0):.2f} ms")
    print(f"   marks: set-state end {1e3*(t1-t0):.3f}, run end "
          f"{1e3*(t2-t0):.3f}")
    for at, dur, name in sorted(log):
        print(f"   {at:8.3f} +{dur:7.3f}  {name}")
ctl.stop()
