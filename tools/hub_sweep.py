"""Accumulation-variant crossover (AUTO_HUB_ENTRIES): step time
of the deterministic gather, the owner-aggregated atomic kernel and the
per-spring warp-aggregated atomic kernel on
  * config B (100^3 lattice, 26 entries per mass), and
  * hub meshes: H hubs with D spokes each (a spoke mass per spring; the hub
    is m1 of its spokes, so its incidence list holds D entries),
for D in a sweep.  Prints one JSON line per (mesh, variant)."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
sys.path.insert(0, os.path.join(ROOT, "tests"))


def hub_case(hubs, spokes):
    import workloads
    n = hubs * (spokes + 1)
    rng = np.random.default_rng(0)
    pos = np.zeros((n, 3))
    a = np.empty(hubs * spokes, np.int64)
    b = np.empty(hubs * spokes, np.int64)
    for h in range(hubs):
        base = h * (spokes + 1)
        pos[base] = (h * 0.5, 0.0, 0.0)
        d = rng.normal(size=(spokes, 3))
        d /= np.linalg.norm(d, axis=1)[:, None]
        pos[base + 1:base + 1 + spokes] = pos[base] + 0.05 * d
        a[h * spokes:(h + 1) * spokes] = base
        b[h * spokes:(h + 1) * spokes] = base + 1 + np.arange(spokes)
    rest, stiff, diam, mass = workloads.materialize(pos, a, b, 1e5, 1000.0,
                                                    1e-3)
    return workloads.make_case(pos * 1.01, mass, a, b, rest, stiff, diam,
                               (0, 0, -9.81), np.zeros((0, 7)))


def time_variant(case, precision, acc, kernel, steps=200):
    from conftest import case_context
    if kernel:
        os.environ["SL_ATOMIC_KERNEL"] = kernel
    else:
        os.environ.pop("SL_ATOMIC_KERNEL", None)
    ctx = case_context(case, precision)
    c = np.zeros(3, np.int64)
    a = {"gather": 0, "atomic": 1, "auto": 2}[acc]
    t = np.arange(steps + 10) * 1e-5
    ctx.step(t[:10], 1e-5, a, c)
    ctx.step(t[10:], 1e-5, a, c)
    ms = ctx.last_step_ms() / steps
    st = ctx.stats()
    st["launches_per_step"] = st["kernel_launches"]
    ctx.close()
    return ms, st


def main():
    import workloads
    prec = sys.argv[1] if len(sys.argv) > 1 else "fp32"
    meshes = [("B100", workloads.config_b(100), 26)]
    for d in (8, 16, 32, 64, 128, 256, 512, 1024, 4096):
        hubs = max(1, 2_000_000 // d)
        meshes.append((f"hub{d}", hub_case(hubs, d), d))
    for name, case, width in meshes:
        springs = len(case["s_m1"])
        for acc, kernel in (("gather", None), ("atomic", "owner"),
                            ("atomic", "spring"), ("auto", None)):
            ms, st = time_variant(case, prec, acc, kernel)
            print(json.dumps({"mesh": name, "widest": width,
                              "springs": springs, "precision": prec,
                              "variant": acc if not kernel else
                              f"atomic-{kernel}", "us_per_step": 1e3 * ms,
                              "upd_per_s": springs / (ms / 1e3),
                              "step_path": st["step_path"]}), flush=True)
        os.environ.pop("SL_ATOMIC_KERNEL", None)


if __name__ == "__main__":
    main()
