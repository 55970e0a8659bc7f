"""Tiled window kernel (csrc/sl_window.cuh, k_win_tma) -- the fp32
production path for banded meshes -- against the split kernel it replaces
(SL_DISABLE_WIN=1) and against the reference oracle, through the C ABI.

The window kernel reads partner positions from shared-memory copies of each
tile's index windows instead of gathering them from L2, and (k, L0) from a
per-tile material table; the per-mass sums have the split kernel's order, so
the two agree to fp32 rounding on the same inputs (see _both), and both are
held to the reference oracle.  Connectivity (alive / zero-length flags,
counters) must be bit-exact in every case.
"""
import os

import numpy as np
import pytest

import oracle as orc
from conftest import case_context, case_times, load_golden, rel_maxnorm

pytestmark = pytest.mark.gpu

PATH_SPLIT_TMA, PATH_WINDOW_TMA = 4, 5


def _ctx(case, precision="fp32", win=True):
    old = os.environ.get("SL_DISABLE_WIN")
    os.environ["SL_DISABLE_WIN"] = "0" if win else "1"
    try:
        return case_context(case, precision)
    finally:
        if old is None:
            del os.environ["SL_DISABLE_WIN"]
        else:
            os.environ["SL_DISABLE_WIN"] = old


def _run(case, times, dt, win, precision="fp32", kill=None, kill_at=None):
    ctx = _ctx(case, precision, win)
    c = np.zeros(3, np.int64)
    if kill is not None:
        done, err = ctx.step(times[:kill_at], dt, 0, c)
        assert err == 0
        ctx.kill_springs(kill.astype(np.int64))
        done, err = ctx.step(times[kill_at:], dt, 0, c)
    else:
        done, err = ctx.step(times, dt, 0, c)
    st = ctx.stats()
    m, s = len(case["m_mass"]), len(case["s_m1"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    alive = np.zeros(s, np.uint8)
    degen = np.zeros(s, np.uint8)
    ctx.download_springs(alive, degen)
    ctx.close()
    return dict(pos=pos, vel=vel, alive=alive, degen=degen, c=c, err=err,
                path=st["step_path"])


def _both(case, times, dt, **kw):
    w = _run(case, times, dt, True, **kw)
    s = _run(case, times, dt, False, **kw)
    assert w["path"] == PATH_WINDOW_TMA, w["path"]
    assert s["path"] == PATH_SPLIT_TMA, s["path"]
    assert w["err"] == s["err"]
    assert np.array_equal(w["alive"], s["alive"])
    assert np.array_equal(w["degen"], s["degen"])
    assert w["c"].tolist() == s["c"].tolist()
    # same (k, L0) values and summation structure, but the window kernel
    # forms the force scale as k - (k L0)/|d| (one FMA) where the split
    # kernel forms k (|d|^2 r - L0) r: equally rounded (fp32 ulps of k),
    # differently -- both hold the fp32 contract (1e-4 of the reference)
    assert rel_maxnorm(w["pos"], s["pos"]) < 1e-5
    assert rel_maxnorm(w["vel"], s["vel"]) < 1e-4
    return w, s


@pytest.mark.parametrize("name", ["cube10_drop", "cube10_contact",
                                  "lat3_contact_drag", "constraints_contacts",
                                  "topology_edits", "yield_break", "worm",
                                  "actuated_quiescent"])
def test_window_matches_split_kernel(name):
    g = load_golden(name)
    n = min(100, int(g["n_steps"]))
    _both(g, case_times(g)[:n], float(g["dt"]))


def _lattice_case(nx, ny, nz, contact=True, robots=0, worm=False):
    """A builder lattice (or a stack of 5^3 robots) in the golden case
    format: the reference bench recipe (cli.py:263-271), x1.01 stretch,
    bottom layer on a friction ground plane."""
    from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                       ObjectStore, Vec3, engine)
    from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
    st = ObjectStore()
    if robots:
        from paper_1911_10274_b200.actuation import configure_worm
        for r in range(robots):
            body = build_lattice(LatticeSpec(Vec3(0, 0.3 * r, 0), 5, 5, 5,
                                             0.05, Material(1e6, 1000.0)), st)
            if worm:
                configure_worm(body, st)
    else:
        build_lattice(LatticeSpec(Vec3(0, 0, 0), nx, ny, nz, 0.05,
                                  Material(1e5, 1000.0)), st)
    m, s = st.mass_slot_count, st.spring_slot_count
    st._m_pos[:m] *= 1.01
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)] if contact else [])
    case = {k: getattr(st, "_" + k)[:m].copy() for k in
            ("m_pos", "m_vel", "m_acc", "m_fext", "m_load", "m_mass",
             "m_fixed", "m_alive", "m_gen")}
    for k in ("s_m1", "s_m2", "s_m1gen", "s_m2gen", "s_rest", "s_k",
              "s_diam", "s_yield", "s_alive", "s_degen"):
        case[k] = getattr(st, "_" + k)[:s].copy()
    for k in ("mode", "amp", "freq", "off", "per"):
        case["s_" + k] = getattr(st, "_s_act_" + k)[:s].copy()
    planes, balls = engine.flatten_contacts(env)
    case.update(gravity=env.gravity.as_array(), drag=0.0, planes=planes,
                balls=balls, gc_kind=np.zeros(0, np.int8),
                gc_vec=np.zeros((0, 3)), lc_off=np.zeros(m + 1, np.int64),
                lc_kind=np.zeros(0, np.int8), lc_vec=np.zeros((0, 3)))
    return case


@pytest.mark.parametrize("shape", [(17, 9, 13), (30, 30, 30), (12, 40, 7)])
def test_window_lattices_match_split_and_oracle(shape):
    case = _lattice_case(*shape)
    dt, n = 1e-4, 60
    times = np.arange(n, dtype=np.float64) * dt
    w, _ = _both(case, times, dt)
    ref = orc.OracleSim(case, nthreads=orc.max_threads())
    for k in range(n):
        ref.step(float(times[k]), dt)
    assert rel_maxnorm(w["pos"], ref.c["m_pos"]) < 1e-4
    assert rel_maxnorm(w["vel"], ref.c["m_vel"]) < 1e-4
    assert np.array_equal(w["alive"], ref.c["s_alive"])


def test_window_robot_stack_and_kills():
    """Stacked 5^3 robots (config D layout, unactuated) with springs killed
    at a pause point: dead A entries must add exactly nothing."""
    case = _lattice_case(0, 0, 0, robots=9)
    dt, n = 1e-4, 80
    times = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(1)
    kill = np.sort(rng.choice(len(case["s_m1"]), 500, replace=False))
    w, _ = _both(case, times, dt, kill=kill, kill_at=30)
    ref = orc.OracleSim(case)
    for k in range(30):
        ref.step(float(times[k]), dt)
    ref.c["s_alive"][kill] = 0
    for k in range(30, n):
        ref.step(float(times[k]), dt)
    assert np.array_equal(w["alive"], ref.c["s_alive"])
    assert rel_maxnorm(w["pos"], ref.c["m_pos"]) < 1e-4
    assert rel_maxnorm(w["vel"], ref.c["m_vel"]) < 1e-4


def test_window_actuated_robot_swarm():
    """Config D shape: worm-actuated 5^3 robots.  The window kernel's
    per-tile actuation table (factor computed once per material per step in
    fp64, kernels.py:55-62) against the split kernel and the oracle over a
    100-step horizon."""
    case = _lattice_case(0, 0, 0, robots=12, worm=True)
    assert (case["s_mode"] == 1).any()
    dt, n = 1e-4, 100
    times = np.arange(n, dtype=np.float64) * dt
    w, _ = _both(case, times, dt)
    ref = orc.OracleSim(case)
    for k in range(n):
        ref.step(float(times[k]), dt)
    assert rel_maxnorm(w["pos"], ref.c["m_pos"]) < 1e-4
    assert rel_maxnorm(w["vel"], ref.c["m_vel"]) < 1e-4


def test_window_param_edits_match_oracle():
    """sl_write_spring_params at a pause (stiffness / rest length changes,
    sine actuation switched on): the window layout's material and actuation
    tables hold values, so the edit must rebuild them -- the trajectory
    equals the oracle's with the same edits."""
    case = _lattice_case(14, 9, 11)
    dt = 1e-4
    times = np.arange(80, dtype=np.float64) * dt
    rng = np.random.default_rng(2)
    sl = np.sort(rng.choice(len(case["s_m1"]), 400, replace=False))
    rest = case["s_rest"][sl] * 0.98
    k = case["s_k"][sl] * 1.5
    mode = np.where(np.arange(len(sl)) % 2 == 0, 1, 0).astype(np.int8)
    amp = np.full(len(sl), 0.1)
    freq = np.full(len(sl), 30.0)
    off = np.zeros(len(sl))
    per = np.full(len(sl), 0.5)
    ctx = _ctx(case)
    c = np.zeros(3, np.int64)
    assert ctx.step(times[:30], dt, 0, c)[1] == 0
    assert ctx.stats()["step_path"] == PATH_WINDOW_TMA
    ctx.write_spring_params(sl, rest, k, case["s_diam"][sl],
                            case["s_yield"][sl], mode, amp, freq, off, per)
    assert ctx.step(times[30:], dt, 0, c)[1] == 0
    assert ctx.stats()["step_path"] == PATH_WINDOW_TMA
    m = len(case["m_mass"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    ctx.close()
    ref = orc.OracleSim(case)
    for n in range(30):
        ref.step(float(times[n]), dt)
    for key, val in (("s_rest", rest), ("s_k", k), ("s_mode", mode),
                     ("s_amp", amp), ("s_freq", freq), ("s_off", off),
                     ("s_per", per)):
        ref.c[key][sl] = val
    for n in range(30, 80):
        ref.step(float(times[n]), dt)
    assert rel_maxnorm(pos, ref.c["m_pos"]) < 1e-4
    assert rel_maxnorm(vel, ref.c["m_vel"]) < 1e-4


@pytest.mark.parametrize("name", ["cube10_drop", "cube10_contact",
                                  "lat3_contact_drag", "constraints_contacts",
                                  "topology_edits"])
def test_window_mixed_matches_split_kernel(name):
    """precision="mixed" (fp64 state and force arithmetic, fp32 (k, L0)):
    the window kernel's fp64 windows and (k, L0) material table give the
    split kernel's forces to fp64 rounding -- the 1e-9 bar of the mixed
    mode's split-vs-exact test (test_gpu_split.py)."""
    g = load_golden(name)
    n = min(100, int(g["n_steps"]))
    t, dt = case_times(g)[:n], float(g["dt"])
    w = _run(g, t, dt, True, precision="mixed")
    s = _run(g, t, dt, False, precision="mixed")
    assert w["path"] == PATH_WINDOW_TMA and s["path"] == PATH_SPLIT_TMA
    assert np.array_equal(w["alive"], s["alive"])
    assert w["c"].tolist() == s["c"].tolist()
    assert rel_maxnorm(w["pos"], s["pos"]) < 1e-9
    assert rel_maxnorm(w["vel"], s["vel"]) < 1e-6


def test_window_exact_fp64_bitwise_equals_exact_kernel():
    """fp64 parity mode on the window layout over the EXACT layout (entries
    in ascending slot order, exact (k, L0) tables, IEEE sqrt / divide):
    bit-identical to the exact TMA kernel (SL_DISABLE_WIN=1) and to the
    oracle, including after kills between launches."""
    case = _lattice_case(20, 17, 9)
    dt, n = 1e-4, 50
    times = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(6)
    kill = np.sort(rng.choice(len(case["s_m1"]), 200, replace=False))
    w = _run(case, times, dt, True, precision="fp64", kill=kill, kill_at=20)
    x = _run(case, times, dt, False, precision="fp64", kill=kill, kill_at=20)
    assert w["path"] == 6 and x["path"] == 2
    assert w["pos"].tobytes() == x["pos"].tobytes()
    assert w["vel"].tobytes() == x["vel"].tobytes()
    ref = orc.OracleSim(case)
    for k in range(n):
        if k == 20:
            ref.c["s_alive"][kill] = 0
        ref.step(float(times[k]), dt)
    assert w["pos"].tobytes() == ref.c["m_pos"].tobytes()
    assert w["vel"].tobytes() == ref.c["m_vel"].tobytes()
