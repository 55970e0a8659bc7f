"""Acceptance run of the reference (pkg/tests/test_acceptance.py:297-326):
a worm-actuated 20x6x6 body crawls for three actuation periods (30,000
steps) through SimController; the reference records a centre-of-mass
displacement of +0.4186 m (pkg/test_output.txt:36) and |dx| < 1e-6 for the
unactuated control."""
import pytest

from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, StepConfig, Vec3)
from paper_1911_10274_b200.actuation import configure_worm
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
from paper_1911_10274_b200.control import SimController

pytestmark = pytest.mark.gpu

RECORDED_DX = 0.4186  # reference run, pkg/test_output.txt:36


def _worm_run(amplitude, precision):
    store = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0), 20, 6, 6, 0.05,
                                     Material(1e6, 1000.0)), store)
    configure_worm(body, store, amplitude=amplitude)
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01,
                      contacts=[ContactPlane(
                          normal=Vec3(0, 0, 1), offset=0.0, stiffness=500.0,
                          static_friction=1.0, kinetic_friction=0.8)])
    ctl = SimController(store, env, StepConfig(dt=1e-4, precision=precision))
    com0 = body.center_of_mass(store).x
    ctl.start(3.0)
    rep = ctl.wait_for_event()
    assert rep.reason == "breakpoint", rep
    assert rep.step_count == 30000
    dx = body.center_of_mass(store).x - com0
    ctl.stop()
    return dx


@pytest.mark.parametrize("precision", ["fp64", "mixed", "fp32"])
def test_worm_locomotion(precision):
    dx = _worm_run(0.2, precision)
    assert dx > 0
    assert abs(dx - RECORDED_DX) < 5e-3 * RECORDED_DX, dx
    assert abs(_worm_run(0.0, precision)) < 1e-6


def _topo_run(replay: bool):
    """Config C (BASELINE.json): the actuated worm with topology edits at
    breakpoints -- every 0.02 s pause, the 30 least-loaded springs are
    removed (cli.py:462-478 rule, loads from the device diagnostics) and 20
    previously removed ones re-added (seeded), through queue_mutations."""
    import numpy as np
    from paper_1911_10274_b200 import engine
    from paper_1911_10274_b200.control import (Breakpoint, CreateSpring,
                                               DeleteSpring)
    orig = engine.DeviceMirror._replay_springs
    if not replay:
        engine.DeviceMirror._replay_springs = lambda self, store, key: False
    try:
        store = ObjectStore()
        body = build_lattice(LatticeSpec(Vec3(0, 0, 0), 20, 6, 6, 0.05,
                                         Material(1e6, 1000.0)), store)
        configure_worm(body, store)
        env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01,
                          contacts=[ContactPlane(
                              normal=Vec3(0, 0, 1), offset=0.0,
                              stiffness=500.0, static_friction=1.0,
                              kinetic_friction=0.8)])
        cfg = StepConfig(dt=1e-4)
        ctl = SimController(store, env, cfg)
        rng = np.random.default_rng(7)
        removed = []
        for k in range(1, 6):
            ctl.set_breakpoint(Breakpoint.at_time(0.02 * k))
        ctl.start(0.1)
        for k in range(5):
            rep = ctl.wait_for_event()
            assert rep.reason == "breakpoint", rep
            loads = engine.device_spring_loads(store, cfg, rep.sim_time, env)
            order = np.argsort(loads.stresses, kind="stable")[:30]
            victims = [h for h, _ in store.iter_springs()]
            slot_to_h = {h.slot: h for h in victims}
            cmds = []
            for slot in loads.slots[order].tolist():
                h = slot_to_h[slot]
                removed.append(store.get_spring(h))
                cmds.append(DeleteSpring(h))
            back = [removed.pop(int(q)) for q in
                    sorted(rng.choice(len(removed), 20, replace=False),
                           reverse=True)]
            cmds += [CreateSpring(sp) for sp in back]
            t = ctl.queue_mutations(cmds)
            assert t.applied
            ctl.start()
        rep = ctl.wait_for_event()
        ctl.stop()
        m = store.mass_slot_count
        mir = engine.mirror_for(store, cfg)
        return (store._m_pos[:m].copy(), store._s_alive[
            :store.spring_slot_count].copy(), getattr(mir, "replays", 0))
    finally:
        engine.DeviceMirror._replay_springs = orig


def test_topology_optimisation_loop_replay_equals_full_upload():
    pos_r, alive_r, replays = _topo_run(True)
    pos_f, alive_f, none = _topo_run(False)
    assert replays >= 3 and none == 0, replays
    assert pos_r.tobytes() == pos_f.tobytes()
    assert (alive_r == alive_f).all()
