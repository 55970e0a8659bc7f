"""SimController on the device: the reference controller's contract
(/root/reference/pkg/tests/test_control.py, control.py:258-650) with the
steps batched into breakpoint-sized launches.

Checked: exact pause steps (at-time rule `bp.time <= now + dt*1e-9`),
state machine errors, pause/resume bitwise transparency, queued mutations
== restart, mutation visibility at step boundaries, snapshots (sync and the
asynchronous pinned-memory variant), numerical abort reporting, and the
whole controller trajectory == the oracle's (fp64, bit for bit).
"""
import threading
import time

import numpy as np
import pytest

import oracle as orc
from paper_1911_10274_b200 import (ContactPlane, ControlStateError,
                                   Environment, Mass, Material, ObjectStore,
                                   Spring, StepConfig, Vec3)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
from paper_1911_10274_b200.control import (Breakpoint, CreateMass,
                                           CreateSpring, DeleteMass,
                                           DeleteSpring, MutationBatch,
                                           SetEnvironment, SetMassField,
                                           SetSpringField, SimController)

pytestmark = pytest.mark.gpu

SOFT = Material(elastic_modulus=1e5, density=1000.0)


def make_lattice(n=3, spacing=0.05, corner=Vec3(0, 0, 0), stretch=None):
    st = ObjectStore()
    body = build_lattice(LatticeSpec(corner=corner, nx=n, ny=n, nz=n,
                                     spacing=spacing, material=SOFT), st)
    if stretch:
        st._m_pos[body.mass_handles.slots] *= stretch
    return st, body


def free_env():
    return Environment(gravity=Vec3(0, 0, 0))


def state_bytes(st):
    n = st.mass_slot_count
    return st._m_pos[:n].tobytes(), st._m_vel[:n].tobytes()


def controller(n=3, dt=1e-4, stretch=1.03, env=None, **kw):
    st, body = make_lattice(n, stretch=stretch)
    return SimController(st, env or free_env(), StepConfig(dt=dt, **kw)), \
        st, body


def test_start_duration_pauses_at_exact_step():
    ctl, *_ = controller(dt=1e-4)
    ctl.start(1.0)
    rep = ctl.wait_for_event(timeout=120)
    assert rep.step_count == 10000 and rep.sim_time == 1.0
    assert rep.reason == "breakpoint"
    assert ctl.device_launches < 200  # batched, not one launch per step
    ctl.stop()


def test_state_machine_errors():
    ctl, *_ = controller()
    with pytest.raises(ControlStateError):
        ctl.pause()
    with pytest.raises(ControlStateError):
        ctl.wait_for_event()
    ctl.start(0.01)
    ctl.wait_for_event()
    ctl.pause()  # already paused: no-op
    ctl.resume()
    with pytest.raises(ControlStateError):
        ctl.resume()
    ctl.stop()
    assert ctl.wait_for_event().state == "done"
    with pytest.raises(ControlStateError):
        ctl.start()


def test_breakpoints_in_order_and_past_breakpoint():
    ctl, *_ = controller(dt=1e-3)
    ctl.set_breakpoint(Breakpoint.at_time(0.5))
    ctl.set_breakpoint(Breakpoint.at_time(0.7))
    ctl.start()
    r1 = ctl.wait_for_event()
    ctl.resume()
    r2 = ctl.wait_for_event()
    assert (r1.step_count, r2.step_count) == (500, 700)
    ctl.set_breakpoint(Breakpoint.at_time(0.05))  # in the past
    ctl.resume()
    assert ctl.wait_for_event().step_count == 700  # fires at once
    ctl.stop()


def test_condition_breakpoint_checks_every_n_steps():
    st, body = make_lattice(3, stretch=1.0, corner=Vec3(0, 0, 0.02))
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.2, contacts=[
        ContactPlane(normal=Vec3(0, 0, 1), offset=0.0, stiffness=500.0,
                     static_friction=0.6, kinetic_friction=0.5)])
    ctl = SimController(st, env, StepConfig(dt=1e-4))
    ctl.set_breakpoint(Breakpoint.on_condition(
        lambda v: v.sim_time > 0.05 and
        np.abs(v.velocities[v.alive]).max() < 5e-3, every=100))
    ctl.start()
    rep = ctl.wait_for_event(timeout=120)
    assert rep.reason == "breakpoint"
    assert rep.breakpoint.kind == "on_condition"
    assert rep.step_count % 100 == 0
    ctl.stop()


def test_concurrent_waiters_and_prompt_pause():
    ctl, *_ = controller(dt=1e-3)
    out = []
    ctl.start(0.2)
    ts = [threading.Thread(target=lambda: out.append(
        ctl.wait_for_event().sim_time)) for _ in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=60)
    assert len(out) == 4 and len(set(out)) == 1
    ctl.resume()
    ctl.pause()
    at = ctl.wait_for_event().step_count
    time.sleep(0.05)
    assert ctl.step_count == at
    ctl.stop()


def test_pause_resume_is_bitwise_transparent():
    c1, s1, _ = controller()
    c1.start(0.1)
    c1.wait_for_event()
    c1.stop()
    c2, s2, _ = controller()
    for _ in range(10):
        c2.start(0.01)
        c2.wait_for_event()
    c2.stop()
    assert state_bytes(s1) == state_bytes(s2)


def test_controller_trajectory_equals_oracle_fp64():
    """1000 controller steps (several launches, time = n*dt) == the
    reference algorithm, bit for bit."""
    st, body = make_lattice(4, stretch=1.04, corner=Vec3(0, 0, -0.01))
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01, contacts=[
        ContactPlane(normal=Vec3(0, 0, 1), offset=0.0, stiffness=800.0,
                     static_friction=0.7, kinetic_friction=0.5)])
    from test_host_parity import our_case
    ref = orc.OracleSim({k: np.array(v) for k, v in our_case(st, env).items()})
    ctl = SimController(st, env, StepConfig(dt=1e-4))
    ctl.set_breakpoint(Breakpoint.at_time(0.0333))
    ctl.start(0.1)
    assert ctl.wait_for_event().step_count == 333
    ctl.resume()
    assert ctl.wait_for_event().step_count == 1000
    ctl.stop()
    ref.run(1000, 1e-4, time_rule="index")
    m = st.mass_slot_count
    assert st._m_pos[:m].tobytes() == ref.c["m_pos"].tobytes()
    assert st._m_vel[:m].tobytes() == ref.c["m_vel"].tobytes()


def test_queued_stiffness_change_matches_restart():
    dt = 1e-4
    ctl, st, body = controller(dt=dt)
    target = body.spring_handles[5]
    ctl.start(0.05)
    ticket = ctl.queue_mutations([SetSpringField(target, "stiffness", 321.0)])
    ctl.wait_for_event()
    assert ticket.resolved and ticket.applied
    snap = ctl.snapshot()
    ctl.start(0.05)
    ctl.wait_for_event()
    ctl.stop()
    direct = state_bytes(st)
    st2, body2 = make_lattice(3, stretch=1.03)
    st2._m_pos[snap.ids] = snap.positions
    st2._m_vel[snap.ids] = snap.velocities
    st2.set_spring_field(body2.spring_handles[5], "stiffness", 321.0)
    c2 = SimController(st2, free_env(), StepConfig(dt=dt))
    c2.start(0.05)
    c2.wait_for_event()
    c2.stop()
    assert state_bytes(st2) == direct


def test_mutation_batches():
    ctl, st, body = controller()
    good, bad = body.mass_handles[1], body.mass_handles[0]
    t = ctl.queue_mutations([SetMassField(good, "m", 9.0)])
    assert t.resolved and t.applied and st.get_mass(good).m == 9.0
    st.delete_mass(bad)
    t = ctl.queue_mutations([SetMassField(good, "m", 5.0),
                             SetMassField(bad, "m", 5.0)])
    assert not t.applied and st.get_mass(good).m == 9.0
    t = ctl.queue_mutations(MutationBatch(
        commands=(SetMassField(good, "m", 5.0), SetMassField(bad, "m", 5.0)),
        policy="partial"))
    assert t.statuses[0] == "applied" and t.statuses[1].startswith("rejected")
    t = ctl.queue_mutations([DeleteMass(bad)])
    assert t.applied and t.statuses[0] == "stale_noop"
    t = ctl.queue_mutations([CreateMass(Mass(pos=Vec3(9, 9, 9), m=1.0))])
    new = t.created_handles[0]
    t2 = ctl.queue_mutations([CreateSpring(Spring(
        m1=body.mass_handles[2], m2=new, rest_length=1.0, stiffness=10.0))])
    assert t2.applied and st.spring_is_live(t2.created_handles[0])
    # the edited topology steps on the device
    ctl.start(0.01)
    ctl.wait_for_event()
    ctl.stop()
    assert np.all(np.isfinite(st._m_pos[:st.mass_slot_count]))


def test_deleted_spring_stays_dead_and_gravity_swap():
    ctl, st, body = controller(stretch=None)
    victim = body.spring_handles[0]
    ctl.start(0.01)
    t = ctl.queue_mutations([DeleteSpring(victim),
                             SetEnvironment(Environment(
                                 gravity=Vec3(0, 0, -1.0)))])
    ctl.wait_for_event()
    assert t.applied and not st.spring_is_live(victim)
    ctl.start(0.01)
    ctl.wait_for_event()
    ctl.stop()
    assert not st.spring_is_live(victim)
    assert np.all(st._m_vel[body.mass_handles.slots][:, 2] < 0)


def test_no_step_observes_partial_batch():
    ctl, st, body = controller(dt=1e-4)
    h0, h1 = body.mass_handles[0], body.mass_handles[1]
    seen = []

    def hook(c):
        seen.append((st._m_mass[h0.slot] == 7.0, st._m_mass[h1.slot] == 7.0))

    ctl.set_step_hook(hook)
    ctl.start(0.02)
    ctl.queue_mutations([SetMassField(h0, "m", 7.0),
                         SetMassField(h1, "m", 7.0)])
    ctl.wait_for_event()
    ctl.start(0.02)
    ctl.wait_for_event()
    ctl.stop()
    assert seen and all(a == b for a, b in seen) and seen[-1] == (True, True)


def test_snapshots_sync_stale_and_async():
    ctl, st, body = controller(dt=1e-3)
    ctl.start(1.0)
    ctl.wait_for_event()
    snap = ctl.snapshot()
    assert snap.sim_time == 1.0 and not snap.stale
    before = snap.positions.copy()
    ctl.start(10.0)
    stale = ctl.snapshot()
    assert stale.stale and np.array_equal(stale.positions, before)
    tk = ctl.snapshot_async()
    assert tk.wait(timeout=60)
    assert tk.step_count >= 1000 and tk.positions.shape[1] == 3
    ctl.pause()
    ctl.wait_for_event()
    ctl.stop()
    assert np.array_equal(snap.positions, before)  # caller-owned copy


def test_async_snapshot_matches_state_at_its_step():
    """The pinned-memory snapshot taken mid-run equals the trajectory of a
    separate run stopped at the snapshot's step."""
    ctl, st, body = controller(dt=1e-4)
    ctl.start(0.2)
    time.sleep(0.01)
    tk = ctl.snapshot_async()
    assert tk.wait(timeout=60)
    ctl.wait_for_event()
    ctl.stop()
    k = tk.step_count
    if k == 0:
        pytest.skip("snapshot resolved before the first launch")
    c2, s2, _ = controller(dt=1e-4)
    c2.start(k * 1e-4)
    assert c2.wait_for_event().step_count == k
    c2.stop()
    m = s2.mass_slot_count
    assert tk.positions[:m].tobytes() == s2._m_pos[:m].tobytes()


def test_numerical_abort_surfaces_in_report():
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1e-30))
    b = st.create_mass(Mass(pos=Vec3(1, 0, 0), m=1e-30))
    st.create_spring(Spring(m1=a, m2=b, rest_length=0.1, stiffness=1e30))
    ctl = SimController(st, free_env(), StepConfig(dt=1.0))
    ctl.start(100.0)
    rep = ctl.wait_for_event(timeout=60)
    assert rep.reason == "error" and rep.error is not None
    assert ctl.state == "done"


def test_pinned_mass_columns_and_lock_time_reads():
    """The mirror moves the mass columns into page-locked memory on first
    push (contents unchanged, growth keeps them pinned); while running,
    store reads see the lock-time state, after the pause the pulled one."""
    from paper_1911_10274_b200 import _native
    ctl, st, body = controller(dt=1e-4)
    h = body.mass_handles[0]
    before = st.get_mass(h).pos.as_array()
    ref_bytes = state_bytes(st)
    ctl.start(10.0)
    for _ in range(20):  # lock-time view, never a half-pulled state
        assert np.array_equal(st.get_mass(h).pos.as_array(), before)
    ctl.pause()
    ctl.wait_for_event(timeout=60)
    assert not np.array_equal(st.get_mass(h).pos.as_array(), before)
    assert state_bytes(st) != ref_bytes
    assert _native.is_pinned(st._m_pos) and _native.is_pinned(st._m_gen)
    grown = st.create_mass(Mass(pos=Vec3(0, 0, 1), m=1.0))
    for _ in range(7):
        st.create_mass(Mass(pos=Vec3(0, 0, 1), m=1.0))
    assert _native.is_pinned(st._m_pos) and st.mass_is_live(grown)
    ctl.stop()


@pytest.mark.parametrize("pinned", [True, False])
def test_apply_snapshot_write_through_matches_full_push(pinned):
    """io.apply_snapshot on a paused controller uploads page-locked
    positions / velocities straight to the device while copying them into
    the store (engine.write_through_begin); the next segment must be bit
    for bit the one a fresh upload of the same state runs."""
    from paper_1911_10274_b200 import _native, engine
    from paper_1911_10274_b200 import io as sio
    ctl, st, _ = controller(n=4, stretch=1.02)
    ctl.start(10 * 1e-4)
    ctl.wait_for_event(timeout=120)
    snap = ctl.snapshot()
    rng = np.random.default_rng(3)
    pos = snap.positions + rng.normal(0, 1e-4, snap.positions.shape)
    vel = snap.velocities + rng.normal(0, 1e-2, snap.velocities.shape)
    if pinned:
        p2, v2 = _native.pinned_empty(pos.shape, np.float64), \
            _native.pinned_empty(vel.shape, np.float64)
        p2[...] = pos
        v2[...] = vel
        pos, vel = p2, v2
    mir = engine.mirror_for(st, ctl._cfg)
    full0 = getattr(mir, "full_pushes", 0)
    sio.apply_snapshot(st, snap.ids, pos, vel)
    if pinned:  # the device already has them: nothing left to send
        assert "_m_pos" not in st.__dict__["_touched"]
    ctl.start(10 * 1e-4)
    ctl.wait_for_event(timeout=120)
    got = ctl.snapshot()
    assert getattr(mir, "full_pushes", 0) == full0
    ctl.stop()
    # the same state through a fresh store / context
    st2, _ = make_lattice(4, stretch=1.02)
    n = st2.mass_slot_count
    st2._m_pos[:n] = np.asarray(pos)
    st2._m_vel[:n] = np.asarray(vel)
    ref = SimController(st2, free_env(), StepConfig(dt=1e-4))
    ref.start(10 * 1e-4)
    ref.wait_for_event(timeout=120)
    want = ref.snapshot()
    ref.stop()
    assert got.positions.tobytes() == want.positions.tobytes()
    assert got.velocities.tobytes() == want.velocities.tobytes()


@pytest.mark.parametrize("touch", [False, True])
def test_pause_pull_fills_snapshot_arena(touch):
    """A pause enqueues the state pull and returns; the next snapshot's
    page-locked arena is filled first (control._pull(pause=True)).  The
    snapshot must equal the store's state, and a host write to the store
    between the pause and the snapshot must show up in it."""
    ctl, st, _ = controller(n=42, stretch=1.01)   # > 65536 masses: arena
    for _ in range(3):
        ctl.start(5 * 1e-4)
        ctl.wait_for_event(timeout=120)
        if touch:
            st._m_pos[7] += 1e-3
        snap = ctl.snapshot()
        n = st.mass_slot_count
        assert snap.positions.tobytes() == st._m_pos[:n].tobytes()
        assert snap.velocities.tobytes() == st._m_vel[:n].tobytes()
        assert np.array_equal(snap.ids, np.arange(n))
    ctl.stop()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_speculative_condition_checks_match_synchronous(precision,
                                                        monkeypatch):
    """Condition breakpoints checked speculatively (the next batch runs
    while the predicate looks at a checkpoint; a hit undoes it, sl_restore)
    pause at the same step with the same state as the synchronous checks
    (reference control.py:579-600): fp64 bit for bit."""
    def run(spec):
        if spec:
            monkeypatch.delenv("SL_NO_SPECULATE", raising=False)
        else:
            monkeypatch.setenv("SL_NO_SPECULATE", "1")
        env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
            normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
            static_friction=1.0, kinetic_friction=0.8)])
        st, _ = make_lattice(n=6, corner=Vec3(0, 0, 0.004))
        ctl = SimController(st, env, StepConfig(dt=1e-4, precision=precision))
        z0 = float(st._m_pos[:st.mass_slot_count, 2].min())
        ctl.set_breakpoint(Breakpoint.on_condition(
            lambda v: float(v.positions[:, 2].min()) < z0 - 2e-4, every=7))
        ctl.start(0.5)
        rep = ctl.wait_for_event(timeout=120)
        snap = ctl.snapshot()
        undos = getattr(ctl, "speculative_undos", 0)
        ctl.stop()
        return rep, snap, undos

    rep_s, snap_s, undos = run(True)
    rep_n, snap_n, _ = run(False)
    assert rep_s.reason == rep_n.reason == "breakpoint"
    assert rep_s.step_count == rep_n.step_count
    assert undos >= 1
    if precision == "fp64":
        assert snap_s.positions.tobytes() == snap_n.positions.tobytes()
        assert snap_s.velocities.tobytes() == snap_n.velocities.tobytes()
    else:
        d = np.abs(snap_s.positions - snap_n.positions).max()
        assert d < 1e-5 * np.abs(snap_n.positions).max()


def test_lock_time_reads_of_deferred_state():
    """With the pause-time pull deferred (store big enough for the snapshot
    arena), lock-time readers during the next run -- a stale snapshot and
    get_mass -- still see the state of the pause (fetched from the stash the
    run kept on the device)."""
    ctl, st, body = controller(n=42, dt=1e-4, stretch=1.01)
    ctl.start(5 * 1e-4)
    ctl.wait_for_event(timeout=120)
    snap = ctl.snapshot()
    h = body.mass_handles[123]
    ctl.start(10.0)
    stale = ctl.snapshot()
    m = st.get_mass(h)
    assert stale.stale
    assert stale.positions.tobytes() == snap.positions.tobytes()
    assert stale.velocities.tobytes() == snap.velocities.tobytes()
    assert np.array_equal(m.pos.as_array(), snap.positions[h.slot])
    ctl.pause()
    ctl.wait_for_event(timeout=120)
    ctl.stop()


def test_apply_snapshot_permuted_rows_after_speculative_upload():
    """io.apply_snapshot starts the write-through before it has checked the
    ids are every slot in order; rows in another order (first and last in
    place) must end up where the ids say, on the host and the device."""
    from paper_1911_10274_b200 import _native
    from paper_1911_10274_b200 import io as sio
    ctl, st, _ = controller(n=4, stretch=1.02)
    ctl.start(5 * 1e-4)
    ctl.wait_for_event(timeout=120)
    snap = ctl.snapshot()
    ids = snap.ids.copy()
    ids[[3, 7]] = ids[[7, 3]]  # swap two rows, ends in place
    pos = _native.pinned_empty(snap.positions.shape, np.float64)
    vel = _native.pinned_empty(snap.velocities.shape, np.float64)
    pos[...] = snap.positions + 1e-4
    vel[...] = snap.velocities
    sio.apply_snapshot(st, ids, pos, vel)
    n = st.mass_slot_count
    want = np.empty((n, 3))
    want[ids] = pos
    assert st._m_pos[:n].tobytes() == want.tobytes()
    ctl.start(5 * 1e-4)
    ctl.wait_for_event(timeout=120)
    got = ctl.snapshot()
    ctl.stop()
    st2, _ = make_lattice(4, stretch=1.02)
    st2._m_pos[:n] = want
    wv = np.empty((n, 3))
    wv[ids] = vel
    st2._m_vel[:n] = wv
    ref = SimController(st2, free_env(), StepConfig(dt=1e-4))
    ref.start(5 * 1e-4)
    ref.wait_for_event(timeout=120)
    exp = ref.snapshot()
    ref.stop()
    assert got.positions.tobytes() == exp.positions.tobytes()


def test_batch_cap_follows_device_time_not_first_batch_wall():
    """A slow first batch (layout build, first touch) must not pin the
    controller at one-step batches: the cap follows the step kernels'
    device time, so it recovers and later segments run as one launch."""
    ctl, st, _ = controller(n=20, stretch=1.01)
    ctl._sec_per_step = 0.05  # as if a 1-step batch had taken 50 ms
    launches = []
    for seg in range(5):
        before = ctl.device_launches
        ctl.start(20 * 1e-4)
        ctl.wait_for_event(timeout=120)
        launches.append(ctl.device_launches - before)
    assert launches[0] > 1 and launches[-2:] == [1, 1], launches
    assert ctl._sec_per_step < 1e-3
    ctl.stop()
