"""Edge cases through the production paths (window / fused kernels, fp32)
and the parity path (fp64): no springs, a single spring, ragged swarms of
bodies of different shapes with isolated masses, mass counts that are not
multiples of 32, a large body next to small ones (fused path ineligible),
all against the reference oracle."""
import numpy as np
import pytest

import oracle as orc
from conftest import case_context, rel_maxnorm
from paper_1911_10274_b200 import (ContactPlane, Environment, Mass, Material,
                                   ObjectStore, Spring, Vec3, engine)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu


def _case(st, env):
    m, s = st.mass_slot_count, st.spring_slot_count
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


def _env():
    return Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])


def _ragged(big=False):
    st = ObjectStore()
    y = 0.0
    shapes = [(3, 3, 3), (4, 5, 2), (40, 1, 1), (2, 2, 2)]
    if big:
        # 1100 masses: one component > 1024 (the fused kernel's largest
        # group), so the per-step window kernel runs
        shapes.insert(1, (11, 10, 10))
    for nx, ny, nz in shapes:
        body = build_lattice(LatticeSpec(Vec3(0, y, 0.01), nx, ny, nz, 0.05,
                                         Material(1e5, 1000.0)), st)
        st._m_pos[body.mass_handles.slots] *= 1.01
        y += 0.05 * ny + 0.2
    for q in range(7):  # isolated masses
        st.create_mass(Mass(pos=Vec3(0.1 * q, y, 0.05), m=1e-3))
    return st


def _run(case, precision, n=60, dt=1e-4):
    ctx = case_context(case, precision)
    c = np.zeros(3, np.int64)
    times = np.arange(n, dtype=np.float64) * dt
    done, err = ctx.step(times, dt, 0, c)
    assert err == 0 and done == n
    st = ctx.stats()
    m = len(case["m_mass"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    ctx.close()
    ref = orc.OracleSim(case)
    for k in range(n):
        ref.step(float(times[k]), dt)
    return pos, vel, ref.c, st


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_no_springs(precision):
    st = ObjectStore()
    for q in range(45):  # not a multiple of 32
        st.create_mass(Mass(pos=Vec3(0.01 * q, 0, 0.02 + 0.001 * q), m=0.1))
    pos, vel, ref, _ = _run(_case(st, _env()), precision)
    tol = 0 if precision == "fp64" else 1e-6
    assert rel_maxnorm(pos, ref["m_pos"]) <= tol
    assert rel_maxnorm(vel, ref["m_vel"]) <= max(tol, 1e-6 * (tol > 0))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_single_spring(precision):
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0.5), m=1.0))
    b = st.create_mass(Mass(pos=Vec3(1.2, 0, 0.5), m=1.0))
    st.create_spring(Spring(m1=a, m2=b, rest_length=1.0, stiffness=100.0))
    pos, vel, ref, _ = _run(_case(st, _env()), precision)
    if precision == "fp64":
        assert pos.tobytes() == ref["m_pos"].tobytes()
    else:
        assert rel_maxnorm(pos, ref["m_pos"]) < 1e-6
        assert rel_maxnorm(vel, ref["m_vel"]) < 1e-4


@pytest.mark.parametrize("big", [False, True])
def test_ragged_swarm(big):
    case = _case(_ragged(big), _env())
    pos, vel, ref, st = _run(case, "fp32")
    # small components only: the fused multi-step kernel; with a 1100-mass
    # body: per-step window kernel
    assert (st["fused_launches"] > 0) == (not big)
    assert rel_maxnorm(pos, ref["m_pos"]) < 1e-4
    assert rel_maxnorm(vel, ref["m_vel"]) < 1e-4
    pos64, vel64, ref64, _ = _run(case, "fp64")
    assert pos64.tobytes() == ref64["m_pos"].tobytes()
    assert vel64.tobytes() == ref64["m_vel"].tobytes()
