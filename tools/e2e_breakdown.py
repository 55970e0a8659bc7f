"""Where the e2e wall time of bench.py config B goes: wraps every method of
the mirror's native Context with a timer, runs the bench's e2e region
(SimController.start / wait_for_event / snapshot) and prints the totals."""
import sys
import time
from collections import defaultdict

sys.argv = [sys.argv[0]] + sys.argv[1:]
sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, engine  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0,
                 accumulation=args.accumulation)
mir = engine.mirror_for(st, cfg)
mir.push(st, env)
mir.ctx.step([0.0, 1e-4, 2e-4], 1e-4, cfg.native_accumulation,
             mir.counters)
mir.ctx.sync()
tot = defaultdict(float)
cnt = defaultdict(int)
ctx = mir.ctx
for name in dir(ctx):
    f = getattr(ctx, name)
    if name.startswith("_") or not callable(f):
        continue

    def wrap(f=f, name=name):
        def g(*a, **k):
            t = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                tot[name] += time.perf_counter() - t
                cnt[name] += 1
        return g
    setattr(ctx, name, wrap())
for rep in range(2):
    tot.clear()
    cnt.clear()
    ctl = SimController(st, env, cfg)
    w0 = time.perf_counter()
    ctl.start(args.steps * 1e-4)
    r = ctl.wait_for_event(timeout=60)
    w1 = time.perf_counter()
    snap = ctl.snapshot()
    w2 = time.perf_counter()
    ctl.stop()
    print(f"rep {rep}: run {1e3*(w1-w0):.1f} ms, snapshot "
          f"{1e3*(w2-w1):.1f} ms, steps {r.step_count}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"  {k:24s} {cnt[k]:4d} calls {1e3*tot[k]:8.2f} ms")

# python-side profile of both threads (controller loop + caller)
import cProfile  # noqa: E402
import pstats  # noqa: E402
orig = SimController._loop
prof_loop = cProfile.Profile()


def loop(self):
    prof_loop.enable()
    try:
        orig(self)
    finally:
        prof_loop.disable()


SimController._loop = loop
w0 = time.perf_counter()
ctl = SimController(st, env, cfg)
ctl.start(args.steps * 1e-4)
ctl.wait_for_event(timeout=60)
w1 = time.perf_counter()
ctl.snapshot()
ctl.stop()
print("profiled run", 1e3 * (w1 - w0), "ms")
print("===== loop thread")
pstats.Stats(prof_loop).sort_stats("cumtime").print_stats(30)
