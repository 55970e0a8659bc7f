"""Engine API on the device: known-answer physics of the reference's engine
tests (/root/reference/pkg/tests/test_engine.py), re-derived and checked
through this package's spring_pass / mass_pass / step / run_steps.

Every call crosses the C ABI into libsoftlat_cuda.so (fp64 parity mode
unless a test says otherwise).
"""
import math

import numpy as np
import pytest

from paper_1911_10274_b200 import (ContactBall, ContactPlane, Environment,
                                   LocalConstraint, Mass, Material,
                                   NumericalAbort, ObjectStore, Spring,
                                   StepConfig, Vec3, engine,
                                   mechanical_energy)
from paper_1911_10274_b200.builder import (LatticeSpec, build_lattice,
                                           derive_spring_constant)

pytestmark = pytest.mark.gpu


def two_masses(x2=2.0, k=100.0, rest=1.0, fixed1=False, **kw):
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0, fixed=fixed1))
    b = st.create_mass(Mass(pos=Vec3(x2, 0, 0), m=1.0))
    s = st.create_spring(Spring(m1=a, m2=b, rest_length=rest, stiffness=k,
                                **kw))
    return st, a, b, s


def free():
    return Environment(gravity=Vec3(0, 0, 0))


@pytest.mark.parametrize("acc", ["linearizable", "atomic"])
@pytest.mark.parametrize("precision", ["fp64", "fp32", "mixed"])
def test_spring_pass_pull_and_rest(acc, precision):
    cfg = StepConfig(dt=1e-4, accumulation=acc, precision=precision)
    st, a, b, _ = two_masses()
    engine.spring_pass(st, 0.0, cfg)
    assert np.allclose(st._m_fext[a.slot], [100, 0, 0], rtol=1e-6)
    assert np.allclose(st._m_fext[b.slot], [-100, 0, 0], rtol=1e-6)
    st, a, b, _ = two_masses(x2=1.0)
    engine.spring_pass(st, 0.0, cfg)
    assert np.all(st._m_fext[:2] == 0)


def test_yield_break_applies_force_then_dies():
    nylon = Material(elastic_modulus=4.56e9, density=1150.0)
    k = derive_spring_constant(nylon, 1e-3, 1e-2)
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    b = st.create_mass(Mass(pos=Vec3(0.012, 0, 0), m=1.0))
    s = st.create_spring(Spring(m1=a, m2=b, rest_length=0.01, stiffness=k,
                                diameter=1e-3, yield_stress=8e7))
    cfg = StepConfig(dt=1e-4)
    engine.spring_pass(st, 0.0, cfg)
    f = float(st._m_fext[a.slot, 0])
    assert f == pytest.approx(k * 0.002, rel=1e-12)
    assert f == pytest.approx(716.0, rel=0.01)
    assert not st.spring_is_live(s)
    st._m_fext[:2] = 0.0
    for _ in range(3):
        engine.spring_pass(st, 0.0, cfg)
        assert np.all(st._m_fext[:2] == 0)


def test_zero_length_spring_is_degenerate_not_broken():
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    b = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    s = st.create_spring(Spring(m1=a, m2=b, rest_length=1.0, stiffness=10.0))
    for precision in ("fp64", "fp32"):
        engine.spring_pass(st, 0.0, StepConfig(dt=1e-4, precision=precision))
        assert np.all(st._m_fext[:2] == 0)
        assert st.spring_is_live(s) and st._s_degen[s.slot]


def test_mass_pass_known_answers():
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    engine.mass_pass(st, Environment(), StepConfig(dt=0.1))
    m = st.get_mass(h)
    assert m.vel.z == pytest.approx(-0.981, rel=1e-12)
    assert m.pos.z == pytest.approx(-0.0981, rel=1e-12)
    assert m.vel.x == m.vel.y == 0.0
    # one-shot f_ext is cleared; load persists
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0, f_ext=Vec3(5, 0, 0)))
    engine.mass_pass(st, free(), StepConfig(dt=0.1))
    assert st.get_mass(h).f_ext == Vec3.zero()
    assert st.get_mass(h).vel.x == pytest.approx(0.5)
    engine.mass_pass(st, free(), StepConfig(dt=0.1))
    assert st.get_mass(h).vel.x == pytest.approx(0.5)
    st.set_applied_load(h, Vec3(2, 0, 0))
    engine.run_steps(st, free(), StepConfig(dt=0.1), 10)
    assert st.get_mass(h).vel.x == pytest.approx(2.5)


def test_fixed_mass_and_drag():
    st, a, b, _ = two_masses(fixed1=True)
    engine.run_steps(st, Environment(), StepConfig(dt=1e-3), 100)
    m = st.get_mass(a)
    assert m.pos == Vec3(0, 0, 0) and m.vel == Vec3.zero()
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3.zero(), m=2.0, vel=Vec3(1, 0, 0)))
    engine.run_steps(st, Environment(gravity=Vec3(0, 0, 0), drag_coeff=0.5),
                     StepConfig(dt=1e-3), 1000)
    assert st.get_mass(h).vel.x == pytest.approx(math.exp(-0.25), rel=1e-3)


def test_local_and_global_constraints():
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3.zero(), m=1.0, local_constraints=(
        LocalConstraint.direction(Vec3(1, 0, 0)),)))
    engine.run_steps(st, Environment(gravity=Vec3(0, 0, -9.81)),
                     StepConfig(dt=1e-3), 100)
    assert st.get_mass(h).pos.z == 0.0 and st.get_mass(h).vel.z == 0.0
    st = ObjectStore()
    hs = [st.create_mass(Mass(pos=Vec3(float(i), 0, 0), m=1.0))
          for i in range(3)]
    st.add_global_constraint(LocalConstraint.plane(Vec3(0, 0, 1)))
    engine.run_steps(st, Environment(), StepConfig(dt=1e-3), 50)
    assert all(st.get_mass(h).pos.z == 0.0 for h in hs)


def test_nan_abort_reports_slot():
    st = ObjectStore()
    good = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    bad = st.create_mass(Mass(pos=Vec3(1, 0, 0), m=1e-30))
    st.create_spring(Spring(m1=good, m2=bad, rest_length=0.1, stiffness=1e30))
    with pytest.raises(NumericalAbort) as ei:
        engine.run_steps(st, free(), StepConfig(dt=1.0), 50)
    assert ei.value.mass_slot == bad.slot


def test_kinetic_friction_stopping_time():
    """mu_k N = 0.5 * 9.81: a 2 m/s block stops after 2/(0.5*9.81) s."""
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3(0, 0, -9.81 / 1e5), m=1.0,
                            vel=Vec3(2, 0, 0)))
    env = Environment(contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=1e5,
        static_friction=0.6, kinetic_friction=0.5)])
    cfg = StepConfig(dt=1e-5)
    steps = 0
    while abs(st.get_mass(h).vel.x) > 1e-3 and steps < 100000:
        engine.run_steps(st, env, cfg, 100, t0=steps * 1e-5)
        steps += 100
    assert steps * 1e-5 == pytest.approx(2.0 / (0.5 * 9.81), rel=0.02)


def test_static_friction_holds_and_ball_pushes():
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3(0, 0, -9.81 / 1e5), m=1.0))
    st.set_applied_load(h, Vec3(1.0, 0, 0))
    env = Environment(contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=1e5,
        static_friction=0.6, kinetic_friction=0.5)])
    engine.run_steps(st, env, StepConfig(dt=1e-4), 1000)
    assert abs(st.get_mass(h).pos.x) < 1e-6
    st = ObjectStore()
    h = st.create_mass(Mass(pos=Vec3(0.95, 0, 0), m=1.0))
    env = Environment(gravity=Vec3(0, 0, 0), contacts=[
        ContactBall(center=Vec3(0, 0, 0), radius=1.0, stiffness=1e3)])
    engine.mass_pass(st, env, StepConfig(dt=1e-3))
    assert st.get_mass(h).acc.x == pytest.approx(50.0)


def test_momentum_and_oscillator_period():
    st, a, b, _ = two_masses()
    engine.step(st, free(), 0.0, StepConfig(dt=1e-4))
    assert np.allclose(st._m_vel[a.slot] + st._m_vel[b.slot], 0, atol=1e-18)
    # fixed-free oscillator, k = 4 pi^2 / 0.1^2: period 0.1 s
    st, a, b, _ = two_masses(x2=1.01, k=3947.84, rest=1.0, fixed1=True)
    env, dt = free(), 1e-5
    e0 = mechanical_energy(st, env).total
    xs, es = [], []
    for n in range(400):  # 4 periods, 100 steps per launch
        engine.run_steps(st, env, StepConfig(dt=dt), 100, t0=n * 100 * dt)
        xs.append(st._m_pos[b.slot, 0] - 1.0)
        es.append(mechanical_energy(st, env).total)
    xs = np.array(xs)
    up = np.flatnonzero((xs[:-1] < 0) & (xs[1:] >= 0))
    cross = (up + 1 - xs[up + 1] / (xs[up + 1] - xs[up])) * 100 * dt
    assert np.diff(cross).mean() == pytest.approx(0.1, rel=5e-3)
    assert (max(es) - min(es)) / e0 < 0.01


def test_barrier_invariant_fused_step():
    """A fused step applies exactly the forces of the pre-step positions:
    spring_pass alone, then mass_pass == one step (bitwise, fp64)."""
    def lat():
        st = ObjectStore()
        build_lattice(LatticeSpec(Vec3(0, 0, 0), 3, 3, 3, 0.05,
                                  Material(1e5, 1000.0)), st)
        st._m_pos[:st.mass_slot_count] *= 1.04
        return st
    cfg = StepConfig(dt=1e-4)
    s1, s2 = lat(), lat()
    engine.run_steps(s1, free(), cfg, 7)
    engine.run_steps(s2, free(), cfg, 7)
    engine.spring_pass(s1, 7e-4, cfg)
    engine.mass_pass(s1, free(), cfg)
    engine.step(s2, free(), 7e-4, cfg)
    n = s1.mass_slot_count
    assert s1._m_pos[:n].tobytes() == s2._m_pos[:n].tobytes()
    assert s1._m_vel[:n].tobytes() == s2._m_vel[:n].tobytes()


def test_step_loop_equals_run_steps():
    """Per-call stepping (host authoritative every step) == one resident
    multi-step launch, bit for bit."""
    def lat():
        st = ObjectStore()
        build_lattice(LatticeSpec(Vec3(0, 0, 0.01), 4, 4, 4, 0.05,
                                  Material(1e5, 1000.0)), st)
        st._m_pos[:st.mass_slot_count] *= 1.03
        return st
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=500.0,
        static_friction=0.6, kinetic_friction=0.5)])
    cfg = StepConfig(dt=1e-4)
    s1, s2 = lat(), lat()
    t = 0.0
    for _ in range(50):
        t = engine.step(s1, env, t, cfg)
    engine.run_steps(s2, env, cfg, 50)
    n = s1.mass_slot_count
    assert s1._m_pos[:n].tobytes() == s2._m_pos[:n].tobytes()
    assert s1._m_vel[:n].tobytes() == s2._m_vel[:n].tobytes()
