"""Who waits for the asynchronous pause pull: prints the stack of every
store._settle that found a pending tail, during steady-state e2e segments
(bench.py config B)."""
import sys
import time
import traceback

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import StepConfig  # noqa: E402
from paper_1911_10274_b200 import io as sio  # noqa: E402
from paper_1911_10274_b200.control import SimController  # noqa: E402
from paper_1911_10274_b200.store import ObjectStore  # noqa: E402

args = bench.parse()
st, env, workload, _, _ = bench.make_workload(args, 0, 1)
cfg = StepConfig(dt=1e-4, precision=args.precision, device=0)
k = args.steps
orig = ObjectStore._settle
log = []


def settle(self):
    if self.__dict__.get("_pending_tail") is not None:
        t = time.perf_counter()
        orig(self)
        log.append((1e3 * (time.perf_counter() - t),
                    "".join(traceback.format_stack(limit=8)[:-1])))
    else:
        orig(self)


ObjectStore._settle = settle
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
    t0 = time.perf_counter()
    sio.apply_snapshot(st, ids, pos_in, vel_in)
    t1 = time.perf_counter()
    ctl.start(k * 1e-4)
    ctl.wait_for_event()
    t2 = time.perf_counter()
    snap = ctl.snapshot()
    t3 = time.perf_counter()
    print(f"rep {rep}: set-state {1e3*(t1-t0):.2f} run {1e3*(t2-t1):.2f} "
          f"snapshot {1e3*(t3-t2):.2f} total {1e3*(t3-t0):.2f} ms")
    for ms, stack in log:
        print(f"  settle waited {ms:.2f} ms at\n{stack}")
ctl.stop()
