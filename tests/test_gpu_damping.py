"""Opt-in spring damping (north_star "Hooke plus damping", spring field
``damping``).  The reference spring is Hooke only
(/root/reference/pkg/src/softlat/kernels.py:66), so:

* c = 0 must leave the reference path bit for bit;
* a damped spring's force on m1 is k(|d| - L0) d^ + c ((v2 - v1) . d^) d^
  (equal and opposite on m2), checked against the analytic damped
  oscillator and against a numpy restatement of one damped step.
"""
import math

import numpy as np
import pytest

import oracle as orc
from conftest import load_golden, rel_maxnorm
from paper_1911_10274_b200 import (Environment, Mass, ObjectStore, Spring,
                                   StepConfig, Vec3, engine)

pytestmark = pytest.mark.gpu


def _oscillator(c, k=50.0, m=0.2, x0=0.01):
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0, fixed=True))
    b = st.create_mass(Mass(pos=Vec3(1.0 + x0, 0, 0), m=m))
    st.create_spring(Spring(m1=a, m2=b, rest_length=1.0, stiffness=k,
                            damping=c))
    return st, b


@pytest.mark.parametrize("precision", ["fp64", "fp32", "mixed"])
@pytest.mark.parametrize("acc", ["gather", "atomic"])
def test_damped_oscillator_known_answer(precision, acc):
    """x'' = -(k/m) x - (c/m) x': amplitude e^{-c t / 2m}, frequency
    sqrt(k/m - (c/2m)^2) (semi-implicit Euler, dt << period)."""
    k, m, c, x0 = 50.0, 0.2, 0.4, 0.01
    st, b = _oscillator(c, k, m, x0)
    dt, n = 1e-5, 40000  # 0.4 s
    cfg = StepConfig(dt=dt, precision=precision, accumulation=acc)
    xs = []
    for _ in range(40):  # no gravity: a pure axial oscillator
        engine.run_steps(st, Environment(gravity=Vec3(0, 0, 0)), cfg,
                         n // 40)
        xs.append(st.get_mass(b).pos.x - 1.0)
    t = np.arange(1, 41) * (n // 40) * dt
    w0 = math.sqrt(k / m)
    g = c / (2 * m)
    wd = math.sqrt(w0 * w0 - g * g)
    want = x0 * np.exp(-g * t) * (np.cos(wd * t) + g / wd * np.sin(wd * t))
    assert np.abs(np.array(xs) - want).max() < 2e-3 * x0


def test_zero_damping_is_the_reference_path():
    """Every spring created with damping=0 (the default) -- and a context
    that had dampers which were then cleared -- steps the golden case bit
    for bit."""
    from conftest import case_context, case_times
    g = load_golden("cube10_contact")
    ctx = case_context(g, "fp64")
    ctx.set_spring_damping(np.full(len(g["s_m1"]), 0.3))
    ctx.set_spring_damping(np.zeros(len(g["s_m1"])))
    cnt = np.zeros(3, np.int64)
    ctx.step(case_times(g), float(g["dt"]), 0, cnt)
    pos = np.zeros((len(g["m_mass"]), 3))
    ctx.download_masses(pos)
    ctx.close()
    assert pos.tobytes() == g["final_pos"].tobytes()


def _damped_step_numpy(case, damp, dt):
    """One reference step (oracle mass pass) with the damper added to each
    spring's force in the serial slot order (kernels.py:36-76 + damper)."""
    sim = orc.OracleSim(case)
    c = sim.c
    p, v = c["m_pos"], c["m_vel"]
    fext = c["m_fext"]
    for s in range(len(c["s_m1"])):
        if not c["s_alive"][s]:
            continue
        i, j = c["s_m1"][s], c["s_m2"][s]
        dx = p[j, 0] - p[i, 0]
        dy = p[j, 1] - p[i, 1]
        dz = p[j, 2] - p[i, 2]
        len2 = dx * dx + dy * dy + dz * dz
        ln = math.sqrt(len2)
        fmag = c["s_k"][s] * (ln - 1.0 * c["s_rest"][s])
        scale = fmag / ln
        vr = (v[j, 0] - v[i, 0]) * dx + (v[j, 1] - v[i, 1]) * dy + \
            (v[j, 2] - v[i, 2]) * dz
        scale = scale + damp[s] * vr / len2
        f = np.array([scale * dx, scale * dy, scale * dz])
        fext[i] += f
        fext[j] -= f
    sim.mass_pass(dt)
    return c


@pytest.mark.parametrize("acc", ["gather", "atomic"])
def test_damped_lattice_matches_numpy_restatement(acc):
    rng = np.random.default_rng(3)
    from test_gpu_window import _lattice_case
    case = _lattice_case(4, 3, 5)
    case["m_vel"] = rng.normal(0, 0.05, case["m_vel"].shape)
    damp = rng.uniform(0, 0.02, len(case["s_m1"]))
    damp[::4] = 0.0
    from conftest import case_context
    dt = 1e-4
    ctx = case_context(case, "fp64")
    ctx.set_spring_damping(damp)
    cnt = np.zeros(3, np.int64)
    ctx.step(np.array([0.0]), dt, 0 if acc == "gather" else 1, cnt)
    m = len(case["m_mass"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    ctx.close()
    ref = _damped_step_numpy(case, damp, dt)
    assert rel_maxnorm(pos, ref["m_pos"]) < 1e-14
    assert rel_maxnorm(vel, ref["m_vel"]) < 1e-12


def test_damped_store_api_precisions_agree():
    """Spring.damping through the store / engine API: fp32 and mixed stay
    within 1e-4 of fp64 over 100 steps of a damped, stretched lattice."""
    from paper_1911_10274_b200 import ContactPlane, Material
    from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

    def make():
        st = ObjectStore()
        body = build_lattice(LatticeSpec(Vec3(0, 0, 0), 6, 5, 7, 0.05,
                                         Material(1e5, 1000.0)), st)
        st._m_pos[body.mass_handles.slots] *= 1.01
        for i, h in enumerate(body.spring_handles):
            st.set_spring_field(h, "damping", 2e-4 * (1 + i % 3))
        return st
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    out = {}
    for prec in ("fp64", "fp32", "mixed"):
        st = make()
        engine.run_steps(st, env, StepConfig(dt=1e-4, precision=prec), 100)
        m = st.mass_slot_count
        out[prec] = (st._m_pos[:m].copy(), st._m_vel[:m].copy())
        # the damper does work: damped != undamped
    st0 = make()
    for h, _ in list(st0.iter_springs()):
        st0.set_spring_field(h, "damping", 0.0)
    engine.run_steps(st0, env, StepConfig(dt=1e-4), 100)
    m = st0.mass_slot_count
    assert rel_maxnorm(st0._m_vel[:m], out["fp64"][1]) > 1e-6
    for prec in ("fp32", "mixed"):
        assert rel_maxnorm(out[prec][0], out["fp64"][0]) < 1e-4
        assert rel_maxnorm(out[prec][1], out["fp64"][1]) < 1e-4
