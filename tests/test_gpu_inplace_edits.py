"""O(edits) topology sync on the production layout (split + window, fp32 /
mixed): spring deletes, creations (re-used slots, LIFO) and retunes between
runs are applied to the live device layout in place (sl_write_springs /
sl_write_spring_params -> k_split_insert on the endpoints' free rows + the
window rebuild of the touched tiles) instead of a device re-index.  Each
segment is checked against the oracle started from the host store at that
pause (1e-4 on positions and velocities, identical spring liveness), and
the context must report the edits as in-place with no further layout
build.  Reference semantics: slot reuse store.py:358-370, kernels.py:28-86.
"""
import numpy as np
import pytest

import oracle as orc
from conftest import rel_maxnorm
from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, Spring, StepConfig, Vec3,
                                   engine)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu
DT = 1e-4


def world():
    st = ObjectStore()
    b = build_lattice(LatticeSpec(Vec3(0, 0, -0.002), 14, 12, 11, 0.05,
                                  Material(1e5, 1000.0)), st)
    st._m_pos[b.mass_handles.slots] *= 1.01
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env, b


def case_of(st, env):
    from test_gpu_fuzz_edits import case_of as c
    return c(st, env)


def edit(st, rng, kind, removed):
    """delete: 40 random springs (their endpoint pairs remembered);
    create: 30 springs re-wiring remembered pairs with new parameters (the
    topology-optimisation pattern: the freed rows take them); retune: 10
    live springs' stiffness."""
    springs = [h for h, _ in st.iter_springs()]
    if kind == "delete":
        for q in rng.choice(len(springs), 40, replace=False):
            sp = st.get_spring(springs[q])
            removed.append((sp.m1, sp.m2))
            st.delete_spring(springs[q])
    elif kind == "create":
        for q in rng.choice(len(removed), 30, replace=False):
            ha, hb = removed[q]
            pa = st.get_mass(ha).pos.as_array()
            pb = st.get_mass(hb).pos.as_array()
            d = float(np.linalg.norm(pb - pa))
            st.create_spring(Spring(m1=ha, m2=hb, rest_length=d * 1.01,
                                    stiffness=float(rng.uniform(500, 3000))))
        removed.clear()
    elif kind == "retune":
        for q in rng.choice(len(springs), 10, replace=False):
            st.set_spring_field(springs[q], "stiffness",
                                float(rng.uniform(100, 900)))


@pytest.mark.parametrize("precision", ["fp32", "mixed", "fp64"])
def test_edits_apply_in_place(precision):
    rng = np.random.default_rng(7)
    st, env, body = world()
    cfg = StepConfig(dt=DT, precision=precision)
    t = engine.run_steps(st, env, cfg, 10)
    mir = engine.mirror_for(st, cfg)
    st0 = mir.ctx.stats()
    assert st0["step_path"] in (5, 6), st0  # the window kernel
    removed = []
    for kind in ("delete", "create", "retune", "delete", "create"):
        edit(st, rng, kind, removed)
        case = case_of(st, env)
        n = 25
        times = engine.step_times(n + 1, DT, t, "accumulate")
        t_next = engine.run_steps(st, env, cfg, n, t0=t)
        ref = orc.OracleSim(case)
        for k in range(n):
            assert ref.step(float(times[k]), DT) == 0
        m, s = st.mass_slot_count, st.spring_slot_count
        st.reconcile_spring_deaths()
        assert np.array_equal(st._s_alive[:s], ref.c["s_alive"]), kind
        if precision == "fp64":  # the exact layout: bit for bit
            assert st._m_pos[:m].tobytes() == ref.c["m_pos"].tobytes(), kind
            assert st._m_vel[:m].tobytes() == ref.c["m_vel"].tobytes(), kind
        else:
            assert rel_maxnorm(st._m_pos[:m], ref.c["m_pos"]) < 1e-4, kind
            assert rel_maxnorm(st._m_vel[:m], ref.c["m_vel"]) < 1e-4, kind
        st._m_pos[:m] = ref.c["m_pos"]
        st._m_vel[:m] = ref.c["m_vel"]
        st._m_acc[:m] = ref.c["m_acc"]
        t = t_next
    sfin = mir.ctx.stats()
    assert sfin["inplace_edits"] == 3, sfin
    # deletes are kills in place; creations / retunes re-wired in place:
    # no device re-index after the first build
    assert sfin["layout_builds"] == st0["layout_builds"], (st0, sfin)


def swarm(n_bodies=24):
    st = ObjectStore()
    bodies = []
    for b in range(n_bodies):
        bodies.append(build_lattice(LatticeSpec(
            Vec3(0.4 * (b % 6), 0.4 * (b // 6), 0.002), 4, 4, 4, 0.05,
            Material(1e5, 1000.0)), st))
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env


def test_edits_apply_in_place_on_fused_bodies():
    """Small bodies run as fused groups (all steps of a call in one launch,
    sl_fused.cuh); deleting and re-adding springs inside a body re-derives
    only its group (k_fused_build over a group list) next to the split /
    window layouts' in-place sync."""
    rng = np.random.default_rng(11)
    st, env = swarm()
    cfg = StepConfig(dt=DT, precision="fp32")
    t = engine.run_steps(st, env, cfg, 10)
    mir = engine.mirror_for(st, cfg)
    s0 = mir.ctx.stats()
    assert s0["fused_groups"] > 0, s0
    removed = []
    for kind in ("delete", "create", "retune", "delete", "create"):
        edit(st, rng, kind, removed)
        case = case_of(st, env)
        n = 30
        times = engine.step_times(n + 1, DT, t, "accumulate")
        f0 = mir.ctx.stats()["fused_launches"]
        t_next = engine.run_steps(st, env, cfg, n, t0=t)
        assert mir.ctx.stats()["fused_launches"] > f0  # still fused
        ref = orc.OracleSim(case)
        for k in range(n):
            assert ref.step(float(times[k]), DT) == 0
        m, s = st.mass_slot_count, st.spring_slot_count
        st.reconcile_spring_deaths()
        assert np.array_equal(st._s_alive[:s], ref.c["s_alive"]), kind
        assert rel_maxnorm(st._m_pos[:m], ref.c["m_pos"]) < 1e-4, kind
        assert rel_maxnorm(st._m_vel[:m], ref.c["m_vel"]) < 1e-4, kind
        st._m_pos[:m] = ref.c["m_pos"]
        st._m_vel[:m] = ref.c["m_vel"]
        st._m_acc[:m] = ref.c["m_acc"]
        t = t_next
    sfin = mir.ctx.stats()
    assert sfin["inplace_edits"] == 3, sfin
    assert sfin["layout_builds"] == s0["layout_builds"], (s0, sfin)
