"""Device diagnostics (sl_energy, sl_spring_loads) against the host numpy
restatement of the reference's engine.mechanical_energy / spring_loads
(engine.py:366-412), on golden states and after device steps."""
import numpy as np
import pytest

from conftest import load_golden
from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, StepConfig, Vec3, engine)
from paper_1911_10274_b200.actuation import configure_worm
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu


def _store(worm=False, n=6):
    st = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0), n, n + 1, n - 1, 0.05,
                                     Material(1e5, 1000.0)), st)
    st._m_pos[body.mass_handles.slots] *= 1.02
    if worm:
        configure_worm(body, st)
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
@pytest.mark.parametrize("worm", [False, True])
def test_device_energy_matches_host(precision, worm):
    st, env = _store(worm)
    cfg = StepConfig(dt=1e-4, precision=precision)
    engine.run_steps(st, env, cfg, 40)  # state now on host and device
    t = 40 * 1e-4
    host = engine.mechanical_energy(st, env, t)
    dev = engine.device_mechanical_energy(st, env, cfg, t, push=False)
    tol = 1e-12 if precision == "fp64" else 1e-5
    for a, b in ((dev.kinetic, host.kinetic),
                 (dev.spring_potential, host.spring_potential),
                 (dev.gravity_potential, host.gravity_potential)):
        assert abs(a - b) <= tol * max(abs(b), 1e-30), (a, b)


@pytest.mark.parametrize("worm", [False, True])
def test_device_spring_loads_match_host(worm):
    st, env = _store(worm)
    cfg = StepConfig(dt=1e-4)  # fp64: exact state on both sides
    engine.run_steps(st, env, cfg, 25)
    # delete a few springs: dead slots are excluded on both sides
    for h, _ in list(st.iter_springs())[3:10]:
        st.delete_spring(h)
    t = 25 * 1e-4
    host = engine.spring_loads(st, t)
    dev = engine.device_spring_loads(st, cfg, t, env)
    assert np.array_equal(dev.slots, host.slots)
    assert np.allclose(dev.lengths, host.lengths, rtol=1e-14, atol=0)
    assert np.allclose(dev.force_magnitudes, host.force_magnitudes,
                       rtol=1e-9, atol=1e-12)
    assert np.array_equal(np.isinf(dev.stresses), np.isinf(host.stresses))
