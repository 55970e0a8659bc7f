"""Random edit sequences through the public store API between device runs
(engine.run_steps, the mirror kept across segments: journal replay, kills,
record writes, mass writes, constraint refreshes), each segment checked
against the oracle started from the host store's arrays at that pause:
fp64 bit-identical positions, velocities and spring flags; fp32 within
tolerance with identical connectivity.  Mass deletes leave springs whose
endpoint died (killed lazily as invalid, kernels.py:37-45); created springs
reuse freed slots (LIFO); parameter edits retune live springs."""
import numpy as np
import pytest

import oracle as orc
from conftest import rel_maxnorm
from paper_1911_10274_b200 import (ContactPlane, Environment, Mass,
                                   Material, ObjectStore, Spring, StepConfig,
                                   Vec3, engine)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
from paper_1911_10274_b200.core import LocalConstraint

pytestmark = pytest.mark.gpu

DT = 1e-4


def world(seed):
    st = ObjectStore()
    b = build_lattice(LatticeSpec(Vec3(0, 0, -0.004), 6, 5, 4, 0.05,
                                  Material(1e5, 1000.0)), st)
    st._m_pos[b.mass_handles.slots] *= 1.01
    build_lattice(LatticeSpec(Vec3(0.5, 0, 0.1), 3, 3, 3, 0.05,
                              Material(2e5, 800.0)), st)
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env


def case_of(st, env):
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
    gk, gv = engine.global_constraint_arrays(st)
    lo, lk, lv = engine.local_constraint_csr(st)
    case.update(gravity=env.gravity.as_array(), drag=env.drag_coeff,
                planes=planes, balls=balls, gc_kind=gk, gc_vec=gv,
                lc_off=lo, lc_kind=lk, lc_vec=lv)
    return case


def live_masses(st):
    return [h for h, _ in st.iter_masses()]


def edit(st, rng):
    ms = live_masses(st)
    springs = [h for h, _ in st.iter_springs()]
    for _ in range(int(rng.integers(3, 8))):
        op = int(rng.integers(0, 8))
        if op == 0 and springs:  # delete springs
            for q in rng.choice(len(springs), min(6, len(springs)),
                                replace=False):
                st.delete_spring(springs[q])
            springs = [h for h, _ in st.iter_springs()]
        elif op == 1:  # new springs between live masses (slot reuse)
            for _ in range(5):
                a, b = rng.choice(len(ms), 2, replace=False)
                pa = st.get_mass(ms[a]).pos.as_array()
                pb = st.get_mass(ms[b]).pos.as_array()
                d = float(np.linalg.norm(pb - pa))
                if d > 0:
                    st.create_spring(Spring(
                        m1=ms[a], m2=ms[b], rest_length=d * 1.02,
                        stiffness=float(rng.uniform(100, 2000))))
            springs = [h for h, _ in st.iter_springs()]
        elif op == 2 and springs:  # retune
            h = springs[int(rng.integers(len(springs)))]
            st.set_spring_field(h, "stiffness", float(rng.uniform(50, 900)))
            h = springs[int(rng.integers(len(springs)))]
            st.set_spring_field(h, "rest_length",
                                st.get_spring(h).rest_length * 0.98)
        elif op == 3 and len(ms) > 10:  # delete a mass (springs go invalid)
            h = ms.pop(int(rng.integers(len(ms))))
            st.delete_mass(h)
        elif op == 4:  # a new mass tied to two live ones
            a, b = rng.choice(len(ms), 2, replace=False)
            p = 0.5 * (st.get_mass(ms[a]).pos.as_array() +
                       st.get_mass(ms[b]).pos.as_array()) + 0.01
            h = st.create_mass(Mass(pos=Vec3(*p), m=0.02))
            for o in (ms[a], ms[b]):
                d = float(np.linalg.norm(st.get_mass(o).pos.as_array() - p))
                st.create_spring(Spring(m1=h, m2=o, rest_length=d,
                                        stiffness=300.0))
            ms.append(h)
        elif op == 5:  # mass fields
            h = ms[int(rng.integers(len(ms)))]
            st.set_mass_field(h, "vel", Vec3(*rng.normal(0, 0.1, 3)))
            h = ms[int(rng.integers(len(ms)))]
            st.set_mass_field(h, "m", float(rng.uniform(0.01, 0.2)))
            h = ms[int(rng.integers(len(ms)))]
            st.set_mass_field(h, "fixed", bool(rng.random() < 0.5))
        elif op == 6:  # local constraints on / off
            h = ms[int(rng.integers(len(ms)))]
            c = LocalConstraint.plane(Vec3(*rng.normal(size=3))) \
                if rng.random() < 0.7 else None
            st.set_mass_field(h, "local_constraints", [c] if c else [])
        elif op == 7:  # persistent load
            h = ms[int(rng.integers(len(ms)))]
            st.set_applied_load(h, Vec3(*rng.normal(0, 0.2, 3)))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_random_edits_between_runs(seed, precision):
    rng = np.random.default_rng(seed)
    st, env = world(seed)
    cfg = StepConfig(dt=DT, precision=precision)
    t = 0.0
    for seg in range(6):
        n = int(rng.integers(5, 40))
        case = case_of(st, env)
        times = engine.step_times(n + 1, DT, t, "accumulate")
        t_next = engine.run_steps(st, env, cfg, n, t0=t)
        ref = orc.OracleSim(case)
        for k in range(n):
            assert ref.step(float(times[k]), DT) == 0
        m, s = st.mass_slot_count, st.spring_slot_count
        st.reconcile_spring_deaths()
        assert np.array_equal(st._s_alive[:s], ref.c["s_alive"]), seg
        if precision == "fp64":
            assert st._m_pos[:m].tobytes() == ref.c["m_pos"].tobytes(), seg
            assert st._m_vel[:m].tobytes() == ref.c["m_vel"].tobytes(), seg
        else:
            assert rel_maxnorm(st._m_pos[:m], ref.c["m_pos"]) < 1e-4, seg
            assert rel_maxnorm(st._m_vel[:m], ref.c["m_vel"]) < 1e-4, seg
            # continue from the reference state so errors do not compound
            st._m_pos[:m] = ref.c["m_pos"]
            st._m_vel[:m] = ref.c["m_vel"]
            st._m_acc[:m] = ref.c["m_acc"]
            st.mass_version += 1
        t = t_next
        edit(st, rng)
