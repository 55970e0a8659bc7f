"""Topology-edit latency on config B (100^3, fp32): delete N springs, run,
re-add N springs on the freed endpoint pairs, run -- wall time of the first
start after each edit (the device sync of the edit + one step) against a
plain one-step start.  Run with SL_NO_INCREMENTAL=1 for the full re-index."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_1911_10274_b200 import Spring, StepConfig, engine  # noqa: E402

st, env = bench.build_workload(100)
cfg = StepConfig(dt=1e-4, precision="fp32")
t = engine.run_steps(st, env, cfg, 5)
mir = engine.mirror_for(st, cfg)
rng = np.random.default_rng(0)


def timed(n=1):
    global t
    w0 = time.perf_counter()
    t = engine.run_steps(st, env, cfg, n, t0=t)
    return 1e3 * (time.perf_counter() - w0)


base = np.median([timed() for _ in range(5)])
for n_edit in (10, 100, 1000):
    springs = [h for h, _ in st.iter_springs()]
    pairs = []
    for q in rng.choice(len(springs), n_edit, replace=False):
        sp = st.get_spring(springs[q])
        pairs.append((sp.m1, sp.m2, sp.rest_length, sp.stiffness))
        st.delete_spring(springs[q])
    b0 = mir.ctx.stats()["layout_builds"]
    t_del = timed()
    for ha, hb, L, k in pairs:
        st.create_spring(Spring(m1=ha, m2=hb, rest_length=L,
                                stiffness=k * 1.1))
    t_add = timed()
    s1 = mir.ctx.stats()
    print(f"{n_edit:5d} edits: delete+step {t_del:7.2f} ms, re-add+step "
          f"{t_add:7.2f} ms (plain step {base:.2f} ms); layout builds "
          f"+{s1['layout_builds'] - b0}, in-place edits {s1['inplace_edits']}")
