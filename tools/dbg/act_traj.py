import os, sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from conftest import case_context, case_times, load_golden, rel_maxnorm
import oracle as orc
name = sys.argv[1] if len(sys.argv) > 1 else "actuated_quiescent"
g = dict(load_golden(name))
times = case_times(g)
def run(prec, split, n):
    os.environ["SL_DISABLE_SPLIT"] = "0" if split else "1"
    ctx = case_context(g, prec)
    c = np.zeros(3, np.int64)
    ctx.step(times[:n], float(g["dt"]), 0, c)
    m = len(g["m_mass"]); p = np.zeros((m, 3)); v = np.zeros((m, 3))
    ctx.download_masses(p, v); ctx.close()
    return p, v
case = {k: g[k] for k in orc.CASE_MASS_KEYS + orc.CASE_SPRING_KEYS + orc.CASE_ENV_KEYS if k in g}
for n in (10, 20, 40, 60, 80, 100):
    ref = orc.OracleSim(case)
    for k in range(n):
        ref.step(float(times[k]), float(g["dt"]))
    rp, rv = ref.c["m_pos"], ref.c["m_vel"]
    row = [n, "|v|max %.3g" % np.abs(rv).max()]
    for prec in ("fp32", "mixed", "fp64"):
        for split in (True, False):
            if prec == "fp64" and split: continue
            p, v = run(prec, split, n)
            row.append("%s%s p%.1e v%.1e" % (prec, "S" if split else "X", rel_maxnorm(p, rp), rel_maxnorm(v, rv)))
    print(*row, flush=True)
