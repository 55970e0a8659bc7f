"""Timeline of bench.py's e2e segment (set-state, K steps, get-state) in
steady state: wall time of each phase and of every native call inside."""
import sys
import time
from collections import defaultdict

sys.argv = [sys.argv[0]] + sys.argv[1:]
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, engine  # noqa: E402
from paper_1911_10274_b200 import io as sio  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0)
k = args.steps
ctl = SimController(st, env, cfg)
ctl.start(k * 1e-4)
ctl.wait_for_event()
warm = ctl.snapshot()
ids = warm.ids.copy()
pos_in = bench._native_pinned_copy(warm.positions)
vel_in = bench._native_pinned_copy(warm.velocities)
mir = engine.mirror_for(st, cfg)
tot = defaultdict(float)
cnt = defaultdict(int)
ctx = mir.ctx
for name in dir(ctx):
    f = getattr(ctx, name)
    if name.startswith("_") or not callable(f):
        continue

    def wrap(f=f, name=name):
        def g(*a, **kw):
            t = time.perf_counter()
            try:
                return f(*a, **kw)
            finally:
                tot[name] += time.perf_counter() - t
                cnt[name] += 1
        return g
    setattr(ctx, name, wrap())
for rep in range(3):
    tot.clear()
    cnt.clear()
    t0 = time.perf_counter()
    sio.apply_snapshot(st, ids, pos_in, vel_in)
    t1 = time.perf_counter()
    ctl.start(k * 1e-4)
    r = ctl.wait_for_event()
    t2 = time.perf_counter()
    snap = ctl.snapshot()
    t3 = time.perf_counter()
    print(f"rep {rep}: set-state {1e3*(t1-t0):.2f} ms, run {1e3*(t2-t1):.2f}"
          f" ms, snapshot {1e3*(t3-t2):.2f} ms, total {1e3*(t3-t0):.2f} ms")
    for name in sorted(tot, key=lambda x: -tot[x]):
        print(f"   {name:20s} {cnt[name]:3d} {1e3*tot[name]:8.2f} ms")
ctl.stop()
