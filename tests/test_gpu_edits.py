"""Topology edits at a pause move only the touched spring records
(DeviceMirror._replay_springs: deletes -> sl_kill_springs in place,
creations into reused slots / field writes -> sl_write_springs, device
re-index).  The trajectory must equal a fresh full upload of the edited
store bit for bit (fp64) and the oracle's."""
import numpy as np
import pytest

import oracle as orc
from conftest import rel_maxnorm
from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, Spring, StepConfig, Vec3,
                                   engine)
from paper_1911_10274_b200.actuation import ActuationParams
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu


def _world():
    st = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0), 7, 6, 5, 0.05,
                                     Material(1e5, 1000.0)), st)
    st._m_pos[body.mass_handles.slots] *= 1.01
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, body, env


def _edit(st, body, rng):
    """delete 40 springs, re-create 25 (LIFO slot reuse), retune 10"""
    handles = [h for h, _ in st.iter_springs()]
    gone = [handles[q] for q in rng.choice(len(handles), 40, replace=False)]
    pairs = [(sp.m1, sp.m2, sp.rest_length, sp.stiffness)
             for sp in (st.get_spring(h) for h in gone)]
    for h in gone:
        st.delete_spring(h)
    for m1, m2, rest, k in pairs[:25]:
        st.create_spring(Spring(m1=m1, m2=m2, rest_length=rest * 0.97,
                                stiffness=k * 1.3))
    live = [h for h, _ in st.iter_springs()]
    for h in [live[q] for q in rng.choice(len(live), 10, replace=False)]:
        st.set_spring_field(h, "actuation", ActuationParams(
            amplitude=0.1, frequency=30.0, period=0.5))


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_replayed_edits_equal_full_upload(precision):
    cfg = StepConfig(dt=1e-4, precision=precision)
    st, body, env = _world()
    engine.run_steps(st, env, cfg, 30)
    mir = engine.mirror_for(st, cfg)
    replays0 = getattr(mir, "replays", 0)
    _edit(st, body, np.random.default_rng(5))
    s_n = st.spring_slot_count
    # the reference: the edited store, uploaded from scratch
    fresh = StepConfig(dt=1e-4, precision=precision, device=0)
    import copy
    st2 = copy.deepcopy(st)
    engine.run_steps(st, env, cfg, 40)
    assert getattr(mir, "replays", 0) == replays0 + 1
    assert st.spring_slot_count == s_n  # the creations reused slots
    engine.run_steps(st2, env, fresh, 40)
    m = st.mass_slot_count
    if precision == "fp64":
        assert st._m_pos[:m].tobytes() == st2._m_pos[:m].tobytes()
        assert st._m_vel[:m].tobytes() == st2._m_vel[:m].tobytes()
    else:
        assert rel_maxnorm(st._m_pos[:m], st2._m_pos[:m]) < 1e-6
    assert np.array_equal(st._s_alive[:s_n], st2._s_alive[:s_n])
