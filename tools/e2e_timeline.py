"""Timeline of one e2e region (bench.py config B): wraps the controller's
and mirror's methods with timestamps and prints when each ran (ms from
start) for a first and a second controller run."""
import sys
import time

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig, engine  # noqa: E402
from paper_1911_10274_b200 import control as C  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0,
                 accumulation=args.accumulation)
mir = engine.mirror_for(st, cfg)
mir.push(st, env)
mir.ctx.step([0.0, 1e-4, 2e-4], 1e-4, cfg.native_accumulation, mir.counters)
mir.ctx.sync()
T0 = [0.0]
log = []


def wrap(obj, name):
    f = getattr(obj, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            log.append((t - T0[0], time.perf_counter() - t, name))
    setattr(obj, name, g)


for n in ("_push", "_pull", "_enter_pause", "_service_snapshots",
          "_steps_to_next_event", "_due_breakpoint", "snapshot", "start",
          "wait_for_event", "__init__", "stop"):
    wrap(C.SimController, n)
for n in ("push", "pull", "set_env"):
    wrap(engine.DeviceMirror, n)
for n in ("upload_masses", "download_masses", "step", "set_local_constraints",
          "set_environment"):
    wrap(mir.ctx, n)
wrap(engine, "local_constraint_csr")
for rep in range(2):
    log.clear()
    T0[0] = time.perf_counter()
    ctl = C.SimController(st, env, cfg)
    ctl.start(args.steps * 1e-4)
    ctl.wait_for_event(timeout=60)
    ctl.snapshot()
    t_end = time.perf_counter() - T0[0]
    ctl.stop()
    print(f"rep {rep}: total {1e3 * t_end:.1f} ms")
    for t, d, n in sorted(log):
        if d > 2e-4:
            print(f"   {1e3 * t:8.2f} +{1e3 * d:7.2f}  {n}")
