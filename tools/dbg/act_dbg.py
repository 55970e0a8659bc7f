import os, sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, "."); sys.path.insert(0, "oracle")
from conftest import case_context, case_times, load_golden, rel_maxnorm

def run(g, prec, split, n):
    os.environ["SL_DISABLE_SPLIT"] = "0" if split else "1"
    ctx = case_context(g, prec)
    c = np.zeros(3, np.int64)
    ctx.step(case_times(g)[:n], float(g["dt"]), 0, c)
    m = len(g["m_mass"]); p = np.zeros((m, 3)); v = np.zeros((m, 3))
    ctx.download_masses(p, v); st = ctx.stats(); ctx.close()
    return p, v, st

base = dict(load_golden("actuated_quiescent"))
variants = {
  "orig": {},
  "all_mode1": {"s_mode": np.where(base["s_mode"] != 0, 1, 0).astype(base["s_mode"].dtype)},
  "all_mode1_off0": {"s_mode": np.where(base["s_mode"] != 0, 1, 0).astype(base["s_mode"].dtype), "s_off": np.zeros_like(base["s_off"])},
  "all_mode1_amp0": {"s_mode": np.where(base["s_mode"] != 0, 1, 0).astype(base["s_mode"].dtype), "s_amp": np.zeros_like(base["s_amp"])},
}
print("modes", np.unique(base["s_mode"], return_counts=True), "per", np.unique(base["s_per"]), "freq", np.unique(base["s_freq"]))
for name, ch in variants.items():
    g = dict(base); g.update(ch)
    for prec in ("fp32", "mixed"):
        for n in (1, 2, 10):
            p1, v1, st = run(g, prec, True, n)
            p2, v2, _ = run(g, prec, False, n)
            d = np.abs(v1 - v2).max(axis=1)
            print(name, prec, n, "pos", rel_maxnorm(p1, p2), "vel", rel_maxnorm(v1, v2), "worst masses", np.argsort(-d)[:5], st if n == 1 else "")
