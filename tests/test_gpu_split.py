"""Split (half-duplex) incidence layout of the tolerance modes vs the exact
layout and vs the reference oracle, through the C ABI.

The split layout (csrc/sl_split.cuh) stores each spring's (k, L0) once and
sums forces in a layout-fixed order, so it is compared within tolerance:
against the exact layout (same precision, SL_DISABLE_SPLIT=1) and against
the fp64 reference (north_star float32 bar, 1e-4 max-norm relative).
Edits (kills between launches) and device-side yield breaks must keep
connectivity bit-exact: the alive flags and counters must equal the
reference's.
"""
import os

import numpy as np
import pytest

import oracle as orc
from conftest import case_context, case_times, load_golden, rel_maxnorm

pytestmark = pytest.mark.gpu


def _ctx(case, precision, split=True):
    old = os.environ.get("SL_DISABLE_SPLIT")
    os.environ["SL_DISABLE_SPLIT"] = "0" if split else "1"
    try:
        return case_context(case, precision)
    finally:
        if old is None:
            del os.environ["SL_DISABLE_SPLIT"]
        else:
            os.environ["SL_DISABLE_SPLIT"] = old


def _state(ctx, case):
    m, s = len(case["m_mass"]), len(case["s_m1"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    alive = np.zeros(s, np.uint8)
    degen = np.zeros(s, np.uint8)
    ctx.download_springs(alive, degen)
    return pos, vel, alive, degen


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
@pytest.mark.parametrize("name", ["cube10_contact", "lat3_contact_drag",
                                  "worm", "constraints_contacts",
                                  "topology_edits", "actuated_quiescent"])
def test_split_matches_exact_layout(name, precision):
    g = load_golden(name)
    n = min(100, int(g["n_steps"]))
    t = case_times(g)[:n]
    out = []
    for split in (True, False):
        ctx = _ctx(g, precision, split)
        c = np.zeros(3, np.int64)
        done, err = ctx.step(t, float(g["dt"]), 0, c)
        assert err == 0 and done == n
        st = ctx.stats()
        out.append((_state(ctx, g), c.copy(), st))
        ctx.close()
    (p1, v1, a1, d1), c1, st1 = out[0]
    (p2, v2, a2, d2), c2, _ = out[1]
    assert np.array_equal(a1, a2) and np.array_equal(d1, d2)
    assert c1.tolist() == c2.tolist()
    tol = 1e-5 if precision == "fp32" else 1e-9
    assert rel_maxnorm(p1, p2) < tol
    assert rel_maxnorm(v1, v2) < 1e3 * tol


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_split_yield_breaks_match_reference(precision):
    """Device-side yield breaks on the split layout: same springs break at
    the same steps as in the reference (connectivity bit-exact), and the
    trajectory stays within the float tolerance."""
    g = load_golden("yield_break")
    ctx = _ctx(g, precision)
    c = np.zeros(3, np.int64)
    done, err = ctx.step(case_times(g), float(g["dt"]), 0, c)
    pos, vel, alive, degen = _state(ctx, g)
    ctx.close()
    assert err == 0 and done == int(g["steps_done"])
    assert np.array_equal(alive, g["final_s_alive"])
    assert c.tolist() == g["final_counters"].tolist()
    assert rel_maxnorm(pos, g["final_pos"]) < 1e-4


@pytest.mark.parametrize("precision", ["fp64", "fp32", "mixed"])
def test_kill_between_launches_matches_oracle(precision):
    """sl_kill_springs at a pause point (delete_spring, store.py:440-458):
    the remaining trajectory equals the oracle's with the same springs
    dead -- bit-exact in fp64 (exact layout), within tolerance otherwise."""
    g = load_golden("cube10_contact")
    t = case_times(g)
    dt = float(g["dt"])
    rng = np.random.default_rng(0)
    kill = np.sort(rng.choice(len(g["s_m1"]), 300, replace=False))
    ref = orc.OracleSim(g)
    ctx = _ctx(g, precision)
    c = np.zeros(3, np.int64)
    ctx.step(t[:60], dt, 0, c)
    for n in range(60):
        ref.step(float(t[n]), dt)
    ctx.kill_springs(kill.astype(np.int64))
    ref.c["s_alive"][kill] = 0
    ctx.step(t[60:120], dt, 0, c)
    for n in range(60, 120):
        ref.step(float(t[n]), dt)
    pos, vel, alive, _ = _state(ctx, g)
    ctx.close()
    assert np.array_equal(alive, ref.c["s_alive"])
    if precision == "fp64":
        assert pos.tobytes() == ref.c["m_pos"].tobytes()
        assert vel.tobytes() == ref.c["m_vel"].tobytes()
    else:
        assert rel_maxnorm(pos, ref.c["m_pos"]) < 1e-4
        assert rel_maxnorm(vel, ref.c["m_vel"]) < 1e-4


def test_split_layout_stats():
    """The split layout streams one (k, L0) per spring: entries counted by
    the library = 32 x (A + B section widths) per slice, and at least two
    incidence entries per alive spring."""
    g = load_golden("cube10_contact")
    ctx = _ctx(g, "fp32")
    c = np.zeros(3, np.int64)
    ctx.step(case_times(g)[:1], float(g["dt"]), 0, c)
    st = ctx.stats()
    ctx.close()
    alive = int(g["s_alive"].sum())
    assert st["entries"] >= 2 * alive
    assert st["slices"] == (len(g["m_mass"]) + 31) // 32
