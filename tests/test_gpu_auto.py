"""accumulation="auto": the deterministic gather, unless the mesh has hub
masses whose incidence lists would serialise one thread per mass -- then
the per-spring atomic variant.  The choice is visible in the
launch count (gather: 1 fused launch per step; atomic: spring + mass)."""
import numpy as np
import pytest

from conftest import rel_maxnorm
from paper_1911_10274_b200 import (Environment, Mass, Material, ObjectStore,
                                   Spring, StepConfig, Vec3, engine)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu


def _star(n=600):
    st = ObjectStore()
    hub = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    rng = np.random.default_rng(4)
    for q in range(n):
        d = rng.normal(size=3)
        d = 0.1 * d / np.linalg.norm(d)
        h = st.create_mass(Mass(pos=Vec3(*(1.05 * d)), m=1e-3))
        st.create_spring(Spring(m1=hub, m2=h, rest_length=0.1,
                                stiffness=50.0))
    return st


def _launches_per_step(st, env, cfg, n=20):
    mir = engine.mirror_for(st, cfg)
    engine.run_steps(st, env, cfg, 2)
    l0 = mir.ctx.stats()["kernel_launches"]
    engine.run_steps(st, env, cfg, n)
    return (mir.ctx.stats()["kernel_launches"] - l0) / n


def test_auto_picks_atomic_for_a_hub_and_gather_for_a_lattice():
    env = Environment(gravity=Vec3(0, 0, 0))
    star = _star()
    ref = _star()
    assert _launches_per_step(star, env,
                              StepConfig(dt=1e-4, accumulation="auto")) >= 2
    engine.run_steps(ref, env, StepConfig(dt=1e-4), 22)  # fp64 gather
    m = star.mass_slot_count
    assert rel_maxnorm(star._m_pos[:m], ref._m_pos[:m]) < 1e-10
    assert rel_maxnorm(star._m_vel[:m], ref._m_vel[:m]) < 1e-6
    lat = ObjectStore()
    build_lattice(LatticeSpec(Vec3(0, 0, 0), 6, 6, 6, 0.05,
                              Material(1e5, 1000.0)), lat)
    cfg = StepConfig(dt=1e-4, accumulation="auto")
    # (+ the per-call state upload kernels)
    assert _launches_per_step(lat, env, cfg) < 1.5
