"""Host-runtime bookkeeping of the lazy pulls (engine._DeferredPull, the
store's settle / stash / overwrite rules) against a stand-in device
context: no GPU needed.  The GPU tests (test_gpu_control.py) run the same
paths on the real library."""
import numpy as np

from paper_1911_10274_b200 import Mass, ObjectStore, Vec3, engine


class FakeCtx:
    """Device state = arrays held here; records the calls."""

    def __init__(self, m):
        self.h = 1
        self.state = {n: np.full((m, 3), float(i + 1))
                      for i, n in enumerate(engine._STATE_NAMES)}
        self.stash = None
        self.calls = []

    def download_masses(self, pos, vel, acc, fext):
        self.calls.append("download")
        for a, n in zip((pos, vel, acc, fext), engine._STATE_NAMES):
            if a is not None:
                a[...] = self.state[n]

    def stash_state(self):
        self.calls.append("stash")
        self.stash = {k: v.copy() for k, v in self.state.items()}

    def download_stash(self, pos, vel, acc, fext):
        self.calls.append("download_stash")
        for a, n in zip((pos, vel, acc, fext), engine._STATE_NAMES):
            if a is not None:
                a[...] = self.stash[n]


def store_with(m=5):
    st = ObjectStore()
    for i in range(m):
        st.create_mass(Mass(pos=Vec3(float(i), 0.0, 0.0), m=1.0))
    return st


def defer(st, ctx, names=engine._STATE_NAMES):
    m = st.mass_slot_count
    d = st.__dict__
    st._defer_state_columns(engine._DeferredPull(
        ctx, {n: d["_c" + n][:m] for n in names}))


def test_first_access_runs_the_deferred_pull():
    st = store_with()
    ctx = FakeCtx(st.mass_slot_count)
    defer(st, ctx)
    assert ctx.calls == []
    pos = st._m_pos[:5]  # tracked access settles
    assert ctx.calls == ["download"]
    assert np.all(pos == 1.0) and np.all(st._m_fext[:5] == 4.0)
    _ = st._m_vel
    assert ctx.calls == ["download"]  # once


def test_overwrite_keeps_the_rest_deferred():
    st = store_with()
    ctx = FakeCtx(st.mass_slot_count)
    defer(st, ctx)
    pos, vel = st._overwrite_state_columns()
    pos[:5] = 9.0
    vel[:5] = 8.0
    assert ctx.calls == []
    assert st._deferred_columns() == ("_m_acc", "_m_fext")
    assert np.all(st._m_acc[:5] == 3.0)  # pulled on access
    assert np.all(st._m_pos[:5] == 9.0)  # not overwritten by the pull
    assert {"_m_pos", "_m_vel"} <= st.__dict__["_touched"]


def test_run_stashes_and_lock_time_readers_fetch_the_stash():
    st = store_with()
    ctx = FakeCtx(st.mass_slot_count)
    defer(st, ctx)
    st.lock_for_run()
    assert ctx.calls == ["stash"]  # no host transfer at start
    ctx.state["_m_pos"][:] = 77.0  # the run moves the device state
    m = st.get_mass(next(h for h, _ in st.iter_masses()))
    assert ctx.calls == ["stash", "download_stash"]
    assert m.pos.as_array()[0] == 1.0  # the lock-time (stashed) state
    st.unlock()


def test_state_epoch_moves_on_every_deferral_and_overwrite():
    st = store_with()
    ctx = FakeCtx(st.mass_slot_count)
    e0 = st.__dict__.get("_state_epoch", 0)
    defer(st, ctx)
    e1 = st.__dict__["_state_epoch"]
    st._overwrite_state_columns()
    assert e0 < e1 < st.__dict__["_state_epoch"]
