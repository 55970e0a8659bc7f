"""Integration engine: the drop-in for the reference's engine module.

Reference: /root/reference/pkg/src/softlat/engine.py.  The public functions
keep their names and signatures (``StepConfig``, ``spring_pass``,
``mass_pass``, ``step``, ``throughput``, diagnostics); the dispatch that
selected numba kernels (engine.py:177-200, 246-250) now drives
libsoftlat_cuda through the C ABI.  ``BACKENDS`` is ``("cuda",)``: there is
no CPU fallback.

Accumulation modes (StepConfig.accumulation):

* ``"linearizable"`` (default) / ``"slotted"`` / ``"gather"`` -- the
  deterministic per-mass gather in ascending spring-slot order.  In fp64 it
  is bit-identical to the reference's serial backend (which is what both
  reference modes compute when run serially, test_engine.py:336-342).
* ``"atomic"`` -- the paper's design (one thread per spring, vector atomics
  into f_ext): order-dependent rounding, tolerance-only.

Precision (StepConfig.precision): ``"fp64"`` (parity), ``"fp32"``,
``"mixed"`` (fp64 mass state, fp32 spring math).

Host arrays are authoritative between calls: ``spring_pass`` / ``mass_pass``
/ ``step`` upload the store, run, and download (exactly the reference's
per-call contract, for tests that poke the arrays between steps).
``run_steps`` and the controller keep the state resident on the device for
many steps and synchronise only at the ends.
"""
from __future__ import annotations

import logging
import math
import weakref
from dataclasses import dataclass

import numpy as np

from . import _native
from .actuation import actuation_factor
from .core import Environment, Mass, Vec3
from .errors import InvalidValueError, NumericalAbort
from .store import ObjectStore

log = logging.getLogger(__name__)

V_STICK = 1e-6                       # engine.py:38
KIND_DIRECTION = 1                   # kernels.py:24-25
KIND_PLANE = 2

# "linearizable" / "slotted" (the reference's names) and "gather" are the
# deterministic per-mass gather; "atomic" the per-spring atomic variant;
# "auto" picks per mesh (gather unless hub masses, sl_api.cu)
ACCUMULATIONS = ("linearizable", "slotted", "gather", "atomic", "auto")
BACKENDS = ("cuda",)
PRECISIONS = ("fp64", "fp32", "mixed")


@dataclass(frozen=True)
class StepConfig:
    """Timestep, accumulation, precision and device (engine.py:44-68)."""

    dt: float
    accumulation: str = "linearizable"
    backend: str = "cuda"
    workers: int | None = None       # accepted for API parity; unused
    precision: str = "fp64"
    device: int = 0
    max_batch: int = 4096            # steps per device launch batch

    def __post_init__(self):
        if not (math.isfinite(self.dt) and self.dt > 0):
            raise InvalidValueError(f"dt must be positive, got {self.dt}")
        if self.accumulation not in ACCUMULATIONS:
            raise InvalidValueError(
                f"accumulation must be one of {ACCUMULATIONS}")
        if self.backend not in BACKENDS:
            raise InvalidValueError(
                f"backend must be one of {BACKENDS} (no CPU fallback)")
        if self.precision not in PRECISIONS:
            raise InvalidValueError(f"precision must be one of {PRECISIONS}")
        if self.workers is not None and self.workers < 1:
            raise InvalidValueError("worker count must be >= 1")
        if self.max_batch < 1:
            raise InvalidValueError("max_batch must be >= 1")

    @property
    def native_accumulation(self) -> int:
        if self.accumulation == "atomic":
            return _native.ACC_ATOMIC
        if self.accumulation == "auto":
            return _native.ACC_AUTO
        return _native.ACC_GATHER


# ----------------------------------------------------------- device mirror
_STATE_NAMES = ("_m_pos", "_m_vel", "_m_acc", "_m_fext")


class _DeferredPull:
    """State columns of a store that only a device holds (after a controller
    pause, or after io.apply_snapshot wrote them straight to the device):
    ``cols`` maps column name -> the store's array.  run() copies them in
    now; stash() -- before the device state changes (lock_for_run) -- keeps
    a device-side copy and returns the pull that reads from it."""

    def __init__(self, ctx, cols: dict, stashed: bool = False):
        self.ctx, self.cols, self.stashed = ctx, dict(cols), stashed

    def _args(self):
        return [self.cols.get(n) for n in _STATE_NAMES]

    def run(self):
        if not self.ctx.h:
            return
        if self.stashed:
            self.ctx.download_stash(*self._args())
        else:
            self.ctx.download_masses(*self._args())

    def stash(self) -> "_DeferredPull":
        if self.stashed or not self.ctx.h:
            return self
        self.ctx.stash_state()
        return _DeferredPull(self.ctx, self.cols, stashed=True)

    def without(self, names) -> "_DeferredPull | None":
        rest = {k: v for k, v in self.cols.items() if k not in names}
        return _DeferredPull(self.ctx, rest, self.stashed) if rest else None


class DeviceMirror:
    """The device-resident copy of one store (the analogue of the reference's
    per-store engine cache, engine.py:71-102), keyed on the store's version
    counters so springs / constraints are re-uploaded only when they change.
    """

    def __init__(self, device: int, precision: str):
        self.ctx = _native.Context(device, precision)
        self._mass_key = None   # (m, host array identity) at the last sync
        self._mass_epoch = -1   # ctx.epoch at the last sync
        self.counters = np.zeros(3, np.int64)
        self._springs_key = None
        self._constraints_key = None
        self._lc_csr = None
        self._custom_slots = np.zeros(0, np.int64)
        self.degen_logged = np.zeros(0, np.bool_)

    # host -> device
    # mass columns by what a host write to them changes on the device
    _STATE_COLS = {"_m_pos", "_m_vel", "_m_acc"}

    def push(self, store: ObjectStore, env: Environment | None,
             masses: bool = True):
        raw = store._raw
        if not _native.is_pinned(store.__dict__["_c_m_pos"]):
            # page-locked mass columns: uploads / pulls at copy-engine speed
            store.adopt_mass_allocator(_native.pinned_empty)
        m, s = store.mass_slot_count, store.spring_slot_count
        touched = store.take_touched()
        full = False  # a whole-column mass upload happened
        if masses or self.ctx.m_n != m:
            # the device holds the host state when nothing but this mirror
            # moved it since the last sync (same arrays, no steps since);
            # then only the columns the host touched travel (raw() -- which
            # waits for copies still landing -- only for columns sent)
            key = (m, store._column_id("_m_pos"))
            synced = (self._mass_key == key and self.ctx.m_n == m and
                      self._mass_epoch == self.ctx.epoch)
            if not synced or touched - self._STATE_COLS:
                self.ctx.upload_masses(*(raw(c)[:m] for c in (
                    "_m_pos", "_m_vel", "_m_acc", "_m_fext", "_m_load",
                    "_m_mass", "_m_fixed", "_m_alive", "_m_gen")))
                self.full_pushes = getattr(self, "full_pushes", 0) + 1
                full = True
            elif touched:
                self.ctx.write_state(
                    *(raw(c)[:m] if c in touched else None
                      for c in ("_m_pos", "_m_vel", "_m_acc")))
            self._mass_key = key
            self._mass_epoch = self.ctx.epoch
        else:  # the caller vouches for the device copy; keep them pending
            store.__dict__["_touched"] |= touched
        key = (s, m, store.topology_version, store.spring_param_version,
               id(store._s_m1))
        if key != self._springs_key and self._replay_springs(store, key):
            pass
        elif key != self._springs_key:
            self.ctx.upload_springs(
                store._s_m1[:s], store._s_m2[:s], store._s_m1gen[:s],
                store._s_m2gen[:s], store._s_rest[:s], store._s_k[:s],
                store._s_diam[:s], store._s_yield[:s], store._s_act_mode[:s],
                store._s_act_amp[:s], store._s_act_freq[:s],
                store._s_act_off[:s], store._s_act_per[:s],
                store._s_alive[:s], store._s_degen[:s])
            self._springs_key = key
            self._journal_at = (store._s_journal_epoch,
                                len(store._s_journal))
            self._custom_slots = np.array(
                sorted(k for k in store._s_custom if k < s), dtype=np.int64)
            self._damp_sent = False  # a full upload clears the dampers
        if store.has_damping and (key != getattr(self, "_damp_key", None)
                                  or not getattr(self, "_damp_sent", False)):
            # opt-in dampers (Spring.damping): the whole column
            self.ctx.set_spring_damping(store._s_damp[:s])
            self._damp_key = key
            self._damp_sent = True
        ckey = (m, store.constraint_version)
        if ckey != self._constraints_key or full:
            # the CSR is rebuilt only when the constraints change; a whole
            # mass upload re-sends the cached one (state-only writes keep
            # the device's constraint flags)
            if ckey != self._constraints_key or self._lc_csr is None:
                self._lc_csr = local_constraint_csr(store)
            self.ctx.set_local_constraints(*self._lc_csr)
            self._constraints_key = ckey
        self.set_env(store, env or Environment())

    def in_sync(self, store: ObjectStore) -> bool:
        """The device holds the host's mass state (same arrays, no device
        steps since the last sync): only host-touched columns differ."""
        m = store.mass_slot_count
        return (self._mass_key == (m, store._column_id("_m_pos")) and
                self.ctx.m_n == m and self._mass_epoch == self.ctx.epoch)

    def _replay_springs(self, store: ObjectStore, key) -> bool:
        """O(edits) spring sync: replay the store's spring journal since the
        last push -- deleted slots become device kills (in place), touched
        live slots whole-record writes (re-indexed on the device) -- when
        the spring arrays are the same allocation and the edit set is small.
        False: the caller uploads everything."""
        old = self._springs_key
        if old is None or old[0] != key[0] or old[1] != key[1] or \
                old[4] != key[4]:
            return False
        epoch, at = getattr(self, "_journal_at", (None, 0))
        if epoch != store._s_journal_epoch or at > len(store._s_journal):
            return False
        pending = store._s_journal[at:]
        if not pending:
            return False
        slots = np.unique(np.concatenate(pending))
        if len(slots) > max(1024, key[0] // 64):
            return False
        alive = store._s_alive[slots].astype(bool)
        dead, live = slots[~alive], slots[alive]
        if len(dead):
            self.ctx.kill_springs(dead)
        if len(live):
            self.ctx.write_springs(
                live, store._s_m1[live], store._s_m2[live],
                store._s_m1gen[live], store._s_m2gen[live],
                store._s_rest[live], store._s_k[live], store._s_diam[live],
                store._s_yield[live], store._s_act_mode[live],
                store._s_act_amp[live], store._s_act_freq[live],
                store._s_act_off[live], store._s_act_per[live],
                store._s_alive[live], store._s_degen[live])
        self._springs_key = key
        self._journal_at = (store._s_journal_epoch, len(store._s_journal))
        self._custom_slots = np.array(
            sorted(k for k in store._s_custom if k < key[0]), dtype=np.int64)
        self.replays = getattr(self, "replays", 0) + 1
        return True

    def set_env(self, store: ObjectStore, env: Environment):
        planes, balls = flatten_contacts(env)
        gk, gv = global_constraint_arrays(store)
        g = np.asarray(env.gravity.as_array(), np.float64)
        key = (g.tobytes(), float(env.drag_coeff), planes.tobytes(),
               balls.tobytes(), gk.tobytes(), gv.tobytes())
        if key == getattr(self, "_env_key", None):
            return  # the device already holds this environment
        self.ctx.set_environment(g, env.drag_coeff, planes, balls, gk, gv,
                                 V_STICK)
        self._env_key = key

    @property
    def has_custom(self) -> bool:
        return len(self._custom_slots) > 0

    def push_custom(self, store: ObjectStore, sim_t: float):
        """engine._fill_custom_factors (engine.py:149-155): callables run on
        the host, factors go to the device."""
        slots = [int(x) for x in self._custom_slots
                 if store._s_alive[x] and x in store._s_actuation]
        if not slots:
            return
        f = [actuation_factor(store._s_actuation[x], sim_t) for x in slots]
        self.ctx.set_custom_factors(np.array(slots, np.int64),
                                    np.array(f, np.float64))

    # device -> host
    def pull(self, store: ObjectStore, springs: bool = True,
             acc: bool = True, fext: bool = True, extra=None) -> bool:
        """Device state into the host store.  ``extra`` = (positions,
        velocities) page-locked (m, 3) buffers (a snapshot's): when given,
        the pull only enqueues -- the extra buffers first, then every store
        column -- and returns True; the store settles on first access and
        the caller waits ctx.download_wait_extra() for the extra buffers."""
        store.materialize_sync()
        m, s = store.mass_slot_count, store.spring_slot_count
        raw = store._raw
        d = store.__dict__
        if extra is not None and m and all(_native.is_pinned(a) for a in (
                *(d["_c" + n] for n in _STATE_NAMES), *extra)):
            # only the extra buffers travel now; the store's state columns
            # stay on the device until the host first needs them
            # (store._settle runs the deferred pull; io.apply_snapshot,
            # rewriting positions / velocities, leaves them there)
            store._drop_deferred()
            cols = {n: d["_c" + n][:m] for n in _STATE_NAMES}
            key = (m, store._column_id("_m_pos"))
            self.ctx.download_state_ex(None, None, None, None,
                                       extra[0], extra[1])
            store._defer_state_columns(_DeferredPull(self.ctx, cols))
            # host == device (deferred): earlier touches are moot
            d["_touched"].difference_update(_STATE_NAMES)
            self._mass_key = key
            self._mass_epoch = self.ctx.epoch
            if springs and s:
                self.ctx.download_springs(store._s_alive[:s].view(np.uint8),
                                          store._s_degen[:s].view(np.uint8))
                store._deaths_maybe = True
            return True
        if acc and fext:
            store._drop_deferred()  # every state column is rewritten below
        if acc and fext and _native.is_pinned(raw("_m_acc")) and \
                _native.is_pinned(raw("_m_fext")):
            # positions / velocities now; accelerations and f_ext keep
            # landing in the page-locked columns while the caller goes on
            # (store._settle waits for them on first access)
            self.ctx.download_state(raw("_m_pos")[:m], raw("_m_vel")[:m],
                                    raw("_m_acc")[:m], raw("_m_fext")[:m])
            ctx = self.ctx
            store.__dict__["_pending_tail"] = \
                lambda: ctx.download_wait() if ctx.h else None
        else:
            self.ctx.download_masses(raw("_m_pos")[:m], raw("_m_vel")[:m],
                                     raw("_m_acc")[:m] if acc else None,
                                     raw("_m_fext")[:m] if fext else None)
        if acc and fext:  # host == device again
            self._mass_key = (m, store._column_id("_m_pos"))
            self._mass_epoch = self.ctx.epoch
        if springs and s:
            self.ctx.download_springs(store._s_alive[:s].view(np.uint8),
                                      store._s_degen[:s].view(np.uint8))
            store._deaths_maybe = True
        return False

    def log_degenerate(self, store: ObjectStore):
        """engine._log_degenerate (engine.py:205-215)."""
        s = store.spring_slot_count
        if len(self.degen_logged) < s:
            grown = np.zeros(s, np.bool_)
            grown[:len(self.degen_logged)] = self.degen_logged
            self.degen_logged = grown
        fresh = np.flatnonzero(store._s_degen[:s] & ~self.degen_logged[:s])
        for slot in fresh.tolist():
            log.warning("spring slot %d has zero length; contributing zero "
                        "force", slot)
        self.degen_logged[fresh] = True


_mirrors: "weakref.WeakKeyDictionary[ObjectStore, dict]" = \
    weakref.WeakKeyDictionary()


def mirror_for(store: ObjectStore, cfg: StepConfig) -> DeviceMirror:
    per = _mirrors.get(store)
    if per is None:
        per = {}
        _mirrors[store] = per
    key = (cfg.device, cfg.precision)
    mir = per.get(key)
    if mir is None:
        mir = DeviceMirror(cfg.device, cfg.precision)
        per[key] = mir
    return mir


def write_through_begin(store: ObjectStore, pos: np.ndarray,
                        vel: np.ndarray) -> list:
    """Start uploading whole position / velocity columns (page-locked,
    (m, 3) fp64) to every mirror of a paused store that holds the rest of
    its state, while the caller copies the same columns into the store
    (io.apply_snapshot).  Returns the mirrors to pass to
    write_through_end."""
    per = _mirrors.get(store)
    if not per or store._locked:
        return []
    if not (_native.is_pinned(pos) and _native.is_pinned(vel)):
        return []
    started = []
    for mir in per.values():
        if mir.in_sync(store):
            mir.ctx.write_state_async(pos, vel, None)
            started.append(mir)
    return started


def write_through_abort(store: ObjectStore, started: list) -> None:
    """write_through_begin's uploads turned out not to apply (the caller's
    rows were not every slot in order): wait for them, and let the next
    start re-send the whole mass state to those mirrors."""
    for mir in started:
        mir.ctx.sync()
        mir._mass_key = None


def write_through_covers(store: ObjectStore, started: list) -> bool:
    """Every mirror of the store took the write-through."""
    return bool(started) and len(started) == len(_mirrors.get(store) or {})


def write_through_end(store: ObjectStore, started: list,
                      host_copied: bool = True) -> None:
    """Wait for write_through_begin's uploads (the caller's arrays are free
    again).  With the host copy done, positions / velocities no longer count
    as host-touched; without it (host_copied False, every mirror covered)
    the store columns are deferred to the first mirror's device copy."""
    for mir in started:
        mir.ctx.sync()
    if not write_through_covers(store, started):
        return
    touched = store.__dict__["_touched"]
    touched.discard("_m_pos")
    touched.discard("_m_vel")
    if not host_copied:
        # positions / velocities plus whatever the store still deferred
        # (the device holds all of it)
        m = store.mass_slot_count
        d = store.__dict__
        names = {"_m_pos", "_m_vel", *store._deferred_columns()}
        store._defer_state_columns(_DeferredPull(
            started[0].ctx, {n: d["_c" + n][:m] for n in names}))


def drop_mirrors(store: ObjectStore):
    """Release the device buffers held for ``store``."""
    if per := _mirrors.get(store):
        if not store._locked:
            store._settle()  # state still only on a device comes home first
    per = _mirrors.pop(store, None)
    for mir in (per or {}).values():
        mir.ctx.close()


# ---------------------------------------------------------------- helpers
def flatten_contacts(env: Environment):
    """planes [P,7] and balls [B,5] exactly as engine.py:223-236 packs
    them."""
    pl = env.planes()
    planes = np.zeros((len(pl), 7))
    for p, c in enumerate(pl):
        planes[p] = (*c.normal.as_tuple(), c.offset, c.stiffness,
                     c.static_friction, c.kinetic_friction)
    bl = env.balls()
    balls = np.zeros((len(bl), 5))
    for b, c in enumerate(bl):
        balls[b] = (*c.center.as_tuple(), c.radius, c.stiffness)
    return planes, balls


def _kind_code(c) -> int:
    return KIND_DIRECTION if c.kind == "direction" else KIND_PLANE


def global_constraint_arrays(store: ObjectStore):
    gc = store.global_constraints
    kinds = np.array([_kind_code(c) for c in gc], dtype=np.int8)
    vecs = (np.array([c.vector.as_tuple() for c in gc], dtype=np.float64)
            .reshape(-1, 3))
    return kinds, vecs


def local_constraint_csr(store: ObjectStore):
    """Per-mass constraint CSR of engine._refresh_constraints
    (engine.py:121-146)."""
    m = store.mass_slot_count
    off = np.zeros(m + 1, dtype=np.int64)
    kinds, vecs = [], []
    for slot in sorted(k for k in store._m_constraints if k < m):
        cs = store._m_constraints[slot]
        off[slot + 1] = len(cs)
        for c in cs:
            kinds.append(_kind_code(c))
            vecs.append(c.vector.as_tuple())
    np.cumsum(off, out=off)
    return (off, np.array(kinds, dtype=np.int8),
            np.array(vecs, dtype=np.float64).reshape(-1, 3))


def _raise_abort(err_slot: int, sim_time: float | None = None):
    slot = err_slot - 1
    raise NumericalAbort(f"non-finite state on mass slot {slot}; "
                         f"reduce dt or stiffness", mass_slot=slot,
                         sim_time=sim_time)


# -------------------------------------------------------- reference API
def spring_pass(store: ObjectStore, sim_t: float, cfg: StepConfig) -> None:
    """Spring forces of all alive springs added into f_ext
    (engine.py:158-202)."""
    mir = mirror_for(store, cfg)
    mir.push(store, None)
    if mir.has_custom:
        mir.push_custom(store, sim_t)
    mir.counters[:] = 0
    mir.ctx.spring_pass(sim_t, cfg.native_accumulation, mir.counters)
    m, s = store.mass_slot_count, store.spring_slot_count
    mir.ctx.download_masses(None, None, None, store._m_fext[:m])
    if s:
        mir.ctx.download_springs(store._s_alive[:s].view(np.uint8),
                                 store._s_degen[:s].view(np.uint8))
        store._deaths_maybe = True
    if mir.counters[2]:
        mir.log_degenerate(store)


def mass_pass(store: ObjectStore, env: Environment, cfg: StepConfig) -> None:
    """Semi-implicit Euler of every alive non-fixed mass; clears f_ext
    (engine.py:218-255)."""
    mir = mirror_for(store, cfg)
    mir.push(store, env)
    err = mir.ctx.mass_pass(cfg.dt)
    mir.pull(store, springs=False)
    if err:
        _raise_abort(err)


def step(store: ObjectStore, env: Environment, sim_t: float,
         cfg: StepConfig) -> float:
    """One fused spring + mass step; returns sim_t + dt
    (engine.py:258-264)."""
    mir = mirror_for(store, cfg)
    mir.push(store, env)
    if mir.has_custom:
        mir.push_custom(store, sim_t)
    mir.counters[:] = 0
    _, err = mir.ctx.step(np.array([sim_t]), cfg.dt, cfg.native_accumulation,
                          mir.counters)
    mir.pull(store, springs=bool(mir.counters[0] or mir.counters[1]
                                 or mir.counters[2]))
    if mir.counters[2]:
        mir.log_degenerate(store)
    if err:
        _raise_abort(err)
    return sim_t + cfg.dt


def step_times(n: int, dt: float, t0: float = 0.0, time_rule: str =
               "accumulate", step0: int = 0) -> np.ndarray:
    """Sim time of each step: ``accumulate`` = repeated ``t += dt``
    (tests/conftest.py:36-41); ``index`` = ``t0 + (step0+k)*dt``
    (control.py:306-307)."""
    if time_rule == "index":
        return t0 + (step0 + np.arange(n, dtype=np.float64)) * dt
    if time_rule != "accumulate":
        raise InvalidValueError(f"unknown time rule {time_rule!r}")
    out = np.empty(n, dtype=np.float64)
    t = float(t0)
    for k in range(n):
        out[k] = t
        t = t + dt
    return out


def run_steps(store: ObjectStore, env: Environment, cfg: StepConfig,
              steps: int, t0: float = 0.0, time_rule: str = "accumulate",
              step0: int = 0) -> float:
    """``steps`` engine steps with the state resident on the device: one
    upload, batched launches, one download.  Same trajectory as calling
    ``step`` in a loop.  Returns the sim time after the last step."""
    times = step_times(steps + 1, cfg.dt, t0, time_rule, step0)
    mir = mirror_for(store, cfg)
    mir.push(store, env)
    counters = np.zeros(3, np.int64)
    done = 0
    err = 0
    while done < steps and not err:
        n = 1 if mir.has_custom else min(cfg.max_batch, steps - done)
        if mir.has_custom:
            mir.push_custom(store, float(times[done]))
        k, err = mir.ctx.step(times[done:done + n], cfg.dt,
                              cfg.native_accumulation, counters)
        done += k
    mir.pull(store, springs=bool(counters.any()))
    if counters[2]:
        mir.log_degenerate(store)
    if err:
        _raise_abort(err)
    return float(times[steps]) if time_rule == "index" else \
        float(times[steps])


def throughput(springs: int, steps: int, wall_seconds: float) -> float:
    """Spring updates per second (engine.py:267-271)."""
    if wall_seconds <= 0:
        raise InvalidValueError("wall_seconds must be positive")
    return springs * steps / wall_seconds


# --------------------------------------------- host diagnostics (numpy)
def check_stability(store: ObjectStore, dt: float,
                    env: Environment | None = None) -> float:
    """dt*sqrt(k_max/m_min), contacts included; warns above 0.5
    (engine.py:274-296).  The spring / mass extrema are masked reductions
    cached on the store's version counters (SimController.start calls this
    on every start: 12.7 M springs made it ~60 ms of host time)."""
    store.reconcile_spring_deaths()
    key = (store.topology_version, store.spring_param_version,
           store.mass_version, store.spring_slot_count,
           store.mass_slot_count)
    cached = getattr(store, "_stability_cache", None)
    if cached is not None and cached[0] == key:
        n_alive, k_springs, m_min = cached[1:]
    else:
        mn, sn = store.mass_slot_count, store.spring_slot_count
        alive = store._m_alive[:mn].astype(bool, copy=False)
        n_alive = int(np.count_nonzero(alive))
        # masked extrema on the host threads (library): the numpy masked
        # reductions took ~14 ms at 12.7 M springs on every new topology
        m_min = _native.masked_extrema(store._m_mass[:mn], alive)[0] \
            if n_alive else np.inf
        k_springs = 0.0
        kc = getattr(store, "_kmax_cache", None)
        kt = store.__dict__.get("_kmax_track")
        if sn and kt is not None and store._s_alive_count > 0:
            # exact through edits (ObjectStore._kmax_add / _kmax_remove)
            k_springs = max(kt[0], 0.0)
        elif sn and kc is not None and kc[0] == (store.topology_version,
                                                 store.spring_param_version,
                                                 sn):
            k_springs = max(kc[1], 0.0) if kc[1] == kc[1] else kc[1]
        elif sn:  # np.max(..., initial=0.0): NaN propagates
            alive_s = store._s_alive[:sn]
            hi = _native.masked_extrema(store._s_k[:sn], alive_s)[1]
            k_springs = hi if (hi != hi or hi > 0.0) else 0.0
            if hi == hi and hi > -np.inf:  # re-seed the tracker
                store.__dict__["_kmax_track"] = [hi, int(np.count_nonzero(
                    (store._s_k[:sn] == hi) & alive_s.astype(bool)))]
        store._stability_cache = (key, n_alive, k_springs, m_min)
    if n_alive == 0:
        return 0.0
    k_max = k_springs
    if env is not None:
        for c in env.contacts:
            k_max = max(k_max, c.stiffness)
    if k_max == 0.0:
        return 0.0
    ratio = dt * math.sqrt(k_max / m_min) if m_min > 0 else math.inf
    if ratio > 0.5:
        log.warning("dt*sqrt(k_max/m_min) = %.3g exceeds 0.5; integration "
                    "may be unstable", ratio)
    return ratio


def contact_forces(mass: Mass, env: Environment) -> Vec3:
    """Contact force on one mass, kernel semantics (engine.py:299-331)."""
    f = mass.f_ext + env.gravity * mass.m - mass.vel * env.drag_coeff
    total = Vec3.zero()
    for pl in env.planes():
        depth = pl.offset - mass.pos.dot(pl.normal)
        if depth <= 0:
            continue
        nmag = pl.stiffness * depth
        normal_force = pl.normal * nmag
        f_now = f + total + normal_force
        v_t = mass.vel - pl.normal * mass.vel.dot(pl.normal)
        f_t = f_now - pl.normal * f_now.dot(pl.normal)
        contrib = normal_force
        tv, tf = v_t.norm(), f_t.norm()
        if tv < V_STICK and tf <= pl.static_friction * nmag:
            contrib = contrib - f_t
        elif tv >= V_STICK:
            contrib = contrib - v_t * (pl.kinetic_friction * nmag / tv)
        elif tf > 0:
            contrib = contrib - f_t * (pl.kinetic_friction * nmag / tf)
        total = total + contrib
    for bl in env.balls():
        d = mass.pos - bl.center
        dist = d.norm()
        depth = bl.radius - dist
        if depth > 0 and dist > 0:
            total = total + d * (bl.stiffness * depth / dist)
    return total


def actuation_factors(store: ObjectStore, sim_t: float,
                      slots: np.ndarray) -> np.ndarray:
    """Vectorised rest-length factors (engine.py:334-352)."""
    mode = store._s_act_mode[slots]
    out = np.ones(len(slots))
    periodic = (mode == 1) | (mode == 2)
    if periodic.any():
        sel = slots[periodic]
        t = (sim_t - store._s_act_off[sel]) % store._s_act_per[sel]
        f = 1.0 + store._s_act_amp[sel] * np.sin(store._s_act_freq[sel] * t)
        quiet = (store._s_act_mode[sel] == 2) & (sim_t < store._s_act_off[sel])
        out[periodic] = np.where(quiet, 1.0, f)
    for idx in np.flatnonzero(mode == 3).tolist():
        out[idx] = actuation_factor(store._s_actuation[int(slots[idx])],
                                    sim_t)
    return out


@dataclass(frozen=True)
class EnergyBreakdown:
    kinetic: float
    spring_potential: float
    gravity_potential: float

    @property
    def total(self) -> float:
        return self.kinetic + self.spring_potential + self.gravity_potential


def mechanical_energy(store: ObjectStore, env: Environment,
                      sim_t: float = 0.0) -> EnergyBreakdown:
    """Kinetic + elastic + gravitational energy (engine.py:366-389)."""
    m = store.alive_mass_slots()
    ke = gpe = 0.0
    if len(m):
        mass = store._m_mass[m]
        vel = store._m_vel[m]
        ke = 0.5 * float(np.sum(mass * np.sum(vel * vel, axis=1)))
        gpe = -float(np.sum(mass * (store._m_pos[m] @ env.gravity.as_array())))
    s = store.alive_spring_slots()
    spe = 0.0
    if len(s):
        d = store._m_pos[store._s_m2[s]] - store._m_pos[store._s_m1[s]]
        lengths = np.linalg.norm(d, axis=1)
        targets = actuation_factors(store, sim_t, s) * store._s_rest[s]
        spe = 0.5 * float(np.sum(store._s_k[s] * (lengths - targets) ** 2))
    return EnergyBreakdown(ke, spe, gpe)


@dataclass(frozen=True)
class SpringLoads:
    slots: np.ndarray
    lengths: np.ndarray
    force_magnitudes: np.ndarray
    stresses: np.ndarray


def device_mechanical_energy(store: ObjectStore, env: Environment,
                             cfg: StepConfig, sim_t: float = 0.0,
                             push: bool = True) -> EnergyBreakdown:
    """mechanical_energy from the device copy of the store (sl_energy): the
    diagnostic cmd_run logs at every pause, without downloading the state.
    ``push=False`` uses the device state as it stands (the store mirror is
    current, e.g. right after engine.run_steps)."""
    mir = mirror_for(store, cfg)
    if push:
        mir.push(store, env)
    if mir.has_custom:
        mir.push_custom(store, sim_t)
    ke, spe, gpe = mir.ctx.energy(sim_t, env.gravity.as_array())
    return EnergyBreakdown(float(ke), float(spe), float(gpe))


def device_spring_loads(store: ObjectStore, cfg: StepConfig,
                        sim_t: float = 0.0, env: Environment | None = None,
                        push: bool = True) -> SpringLoads:
    """spring_loads with the per-spring gather / length / |F| on the device
    (sl_spring_loads); compaction over alive slots and the stress on the
    host, exactly as spring_loads forms them."""
    mir = mirror_for(store, cfg)
    if push:
        mir.push(store, env)
    if mir.has_custom:
        mir.push_custom(store, sim_t)
    n = store.spring_slot_count
    lengths, fmag = mir.ctx.spring_loads(sim_t, n)
    s = store.alive_spring_slots()
    lengths, fmag = lengths[s], fmag[s]
    area = 0.25 * np.pi * store._s_diam[s] ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        stress = np.where(area > 0, fmag / np.where(area > 0, area, 1.0),
                          np.where(fmag > 0, np.inf, 0.0))
    return SpringLoads(s, lengths, fmag, stress)


def spring_loads(store: ObjectStore, sim_t: float = 0.0) -> SpringLoads:
    """Per-spring |F| and stress (engine.py:402-412)."""
    s = store.alive_spring_slots()
    d = store._m_pos[store._s_m2[s]] - store._m_pos[store._s_m1[s]]
    lengths = np.linalg.norm(d, axis=1)
    targets = actuation_factors(store, sim_t, s) * store._s_rest[s]
    fmag = np.abs(store._s_k[s] * (lengths - targets))
    area = 0.25 * np.pi * store._s_diam[s] ** 2
    with np.errstate(divide="ignore", invalid="ignore"):
        stress = np.where(area > 0, fmag / np.where(area > 0, area, 1.0),
                          np.where(fmag > 0, np.inf, 0.0))
    return SpringLoads(s, lengths, fmag, stress)
