"""Where the e2e time of bench config B goes (cProfile of the public-API
run: SimController.start -> wait_for_event -> snapshot)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import bench
from paper_1911_10274_b200 import StepConfig, engine
from paper_1911_10274_b200.control import SimController
st, env = bench.build_workload(100)
cfg = StepConfig(dt=1e-4, precision="fp32")
mir = engine.mirror_for(st, cfg)
mir.push(st, env)
for rep in range(3):
    ctl = SimController(st, env, cfg)
    k = 2000
    pr = cProfile.Profile()
    w0 = time.perf_counter()
    pr.enable()
    ctl.start(k * cfg.dt)
    r = ctl.wait_for_event()
    snap = ctl.snapshot()
    pr.disable()
    wall = time.perf_counter() - w0
    ctl.stop()
    print("rep", rep, "wall", wall)
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
