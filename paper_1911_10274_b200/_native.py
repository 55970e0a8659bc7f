"""ctypes binding of libsoftlat_cuda.so (include/softlat_cuda.h).

This is the only path to the compute: there is no CPU fallback.  Loading
fails loudly if the shared library was not built (run
``python -c "import __graft_entry__ as g; g.build()"`` or
``python paper_1911_10274_b200/_build.py``).
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import (DeviceError, InvalidValueError, NumericalAbort,
                     SoftlatError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsoftlat_cuda.so")

SL_OK, SL_EINVAL, SL_ECUDA, SL_ENUMERIC, SL_ESTATE, SL_EUNSUPPORTED = range(6)
PRECISIONS = {"fp64": 0, "fp32": 1, "mixed": 2}
ACC_GATHER, ACC_ATOMIC, ACC_AUTO = 0, 1, 2

# every symbol the header declares (tests check the .so exports them all)
EXPORTS = (
    "sl_abi_version", "sl_device_count", "sl_create", "sl_destroy",
    "sl_last_error", "sl_get_stats", "sl_upload_masses", "sl_upload_springs",
    "sl_set_environment", "sl_set_local_constraints", "sl_set_custom_factors",
    "sl_write_masses", "sl_write_spring_params", "sl_write_springs",
    "sl_kill_springs", "sl_step",
    "sl_spring_pass", "sl_mass_pass", "sl_download_masses",
    "sl_download_springs", "sl_snapshot_begin", "sl_snapshot_ready",
    "sl_snapshot_wait", "sl_timer_start", "sl_timer_stop", "sl_sync",
    "sl_last_step_ms",
    "sl_step_async", "sl_step_finish", "sl_mark_ghosts", "sl_state_pointers",
    "sl_state_lo", "sl_get_stream", "sl_energy", "sl_spring_loads", "sl_host_alloc",
    "sl_host_free", "sl_format_snapshot", "sl_lattice_counts",
    "sl_build_lattice", "sl_host_fill", "sl_host_copy",
    "sl_host_masked_extrema", "sl_set_spring_damping", "sl_halo_init",
    "sl_halo_local", "sl_halo_ipc_handles", "sl_halo_ipc_open",
    "sl_halo_set_peer", "sl_halo_commit", "sl_write_state",
    "sl_write_state_async",
    "sl_host_is_iota", "sl_download_state", "sl_download_wait",
    "sl_download_state_ex", "sl_download_wait_extra",
    "sl_stash_state", "sl_download_stash", "sl_checkpoint",
    "sl_checkpoint_view_wait", "sl_restore")


class SlStats(C.Structure):
    _fields_ = [("masses", C.c_int64), ("springs", C.c_int64),
                ("alive_springs", C.c_int64), ("entries", C.c_int64),
                ("slices", C.c_int64), ("layout_builds", C.c_int64),
                ("device_bytes", C.c_int64), ("kernel_launches", C.c_int64),
                ("precision", C.c_int32), ("device", C.c_int32),
                ("step_path", C.c_int32), ("split_batch", C.c_int32),
                ("fused_groups", C.c_int64), ("fused_launches", C.c_int64),
                ("fused_aborts", C.c_int64),
                ("win_tile_slices", C.c_int32), ("win_stages", C.c_int32),
                ("inplace_edits", C.c_int64)]

STEP_PATHS = {0: "none", 1: "k_gather_step", 2: "k_gather_tma",
              3: "k_split_step", 4: "k_split_tma", 5: "k_win_tma",
              6: "k_win_tma (exact)"}


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load (once) and declare signatures.  Raises if the .so is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise SoftlatError(
                f"CUDA library not built: {path} is missing; build it with "
                "paper_1911_10274_b200/_build.py (no CPU fallback exists)")
        lib = C.CDLL(path)
        P, I64, D, I = C.c_void_p, C.c_int64, C.c_double, C.c_int
        sig = {
            "sl_abi_version": ([], I),
            "sl_device_count": ([P], I),
            "sl_create": ([I, I, P], I),
            "sl_destroy": ([P], I),
            "sl_last_error": ([P], C.c_char_p),
            "sl_get_stats": ([P, P], I),
            "sl_upload_masses": ([P, I64] + [P] * 9, I),
            "sl_upload_springs": ([P, I64] + [P] * 15, I),
            "sl_set_environment": ([P, P, D, P, I64, P, I64, P, P, I64, D], I),
            "sl_set_local_constraints": ([P, I64, P, P, P, I64], I),
            "sl_set_custom_factors": ([P, I64, P, P], I),
            "sl_write_masses": ([P, I64] + [P] * 10, I),
            "sl_write_spring_params": ([P, I64] + [P] * 10, I),
            "sl_kill_springs": ([P, I64, P], I),
            "sl_write_springs": ([P, I64, P] + [P] * 15, I),
            "sl_step": ([P, I64, P, D, I, P, P, P], I),
            "sl_spring_pass": ([P, D, I, P], I),
            "sl_mass_pass": ([P, D, P], I),
            "sl_download_masses": ([P, P, P, P, P], I),
            "sl_download_springs": ([P, P, P], I),
            "sl_snapshot_begin": ([P], I),
            "sl_snapshot_ready": ([P, P], I),
            "sl_snapshot_wait": ([P, P, P], I),
            "sl_timer_start": ([P], I),
            "sl_timer_stop": ([P, P], I),
            "sl_last_step_ms": ([P, P], I),
            "sl_set_spring_damping": ([P, I64, P], I),
            "sl_halo_init": ([P, I, P], I),
            "sl_halo_local": ([P, P], I),
            "sl_halo_ipc_handles": ([P, P], I),
            "sl_halo_ipc_open": ([P, P, P], I),
            "sl_halo_set_peer": ([P, I, P, I], I),
            "sl_halo_commit": ([P], I),
            "sl_write_state": ([P, I64, P, P, P], I),
            "sl_write_state_async": ([P, I64, P, P, P], I),
            "sl_host_is_iota": ([P, I64, I, P], I),
            "sl_download_state": ([P, P, P, P, P], I),
            "sl_download_wait": ([P], I),
            "sl_download_state_ex": ([P, P, P, P, P, P, P, C.c_int], I),
            "sl_download_wait_extra": ([P], I),
            "sl_stash_state": ([P], I),
            "sl_download_stash": ([P, P, P, P, P], I),
            "sl_checkpoint": ([P, P, P], I),
            "sl_checkpoint_view_wait": ([P], I),
            "sl_restore": ([P], I),
            "sl_sync": ([P], I),
            "sl_step_async": ([P, I64, P, D, I], I),
            "sl_step_finish": ([P, P, P, P], I),
            "sl_mark_ghosts": ([P, I64, P], I),
            "sl_state_pointers": ([P, P, P, P], I),
            "sl_state_lo": ([P, P], I),
            "sl_get_stream": ([P, P], I),
            "sl_energy": ([P, D, P, P], I),
            "sl_spring_loads": ([P, D, P, P], I),
            "sl_host_alloc": ([C.c_size_t, P], I),
            "sl_host_free": ([P], I),
            "sl_format_snapshot": ([I64, P, P, P, I, P, C.c_size_t, P], I),
            "sl_lattice_counts": ([I64, I64, I64, P, P], I),
            "sl_build_lattice": ([I64, I64, I64, P, D, D, D, D, I] + [P] * 6,
                                 I),
            "sl_host_fill": ([P, P, C.c_size_t, I64, I], I),
            "sl_host_copy": ([P, P, C.c_size_t, I], I),
            "sl_host_masked_extrema": ([P, P, I64, I, P, P], I),
        }
        for name, (args, res) in sig.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype, shape_tail=()):
    """Contiguous view/copy with the dtype the ABI expects."""
    arr = np.ascontiguousarray(a, dtype=dtype)
    return arr


def device_count() -> int:
    lib = load_library()
    n = C.c_int(0)
    rc = lib.sl_device_count(C.byref(n))
    return int(n.value) if rc == SL_OK else 0


class _PinnedBlock:
    """Owner of one sl_host_alloc buffer; freed when the last numpy array
    viewing it is collected (the arrays keep it alive through .base)."""

    def __init__(self, nbytes: int):
        lib = load_library()
        p = C.c_void_p()
        if lib.sl_host_alloc(max(1, nbytes), C.byref(p)) != SL_OK:
            raise SoftlatError("sl_host_alloc: " +
                               (lib.sl_last_error(None) or b"").decode())
        self._lib, self.ptr, self.nbytes = lib, p.value, nbytes
        self.__array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "version": 3,
            "data": (p.value, False)}

    def __del__(self):
        if self.ptr:
            self._lib.sl_host_free(C.c_void_p(self.ptr))
            self.ptr = None


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array in page-locked host memory (sl_host_alloc)."""
    dt = np.dtype(dtype)
    n = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    raw = np.asarray(_PinnedBlock(n))
    return raw[:n].view(dt).reshape(shape)


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def host_copy(a: np.ndarray) -> np.ndarray:
    """np.array(a) with the copy (and the fresh pages' first touch) spread
    over the host threads (sl_host_copy); small arrays copy in numpy."""
    if a.nbytes < (1 << 20) or not a.flags.c_contiguous:
        return np.array(a)
    out = np.empty_like(a)
    rc = load_library().sl_host_copy(_ptr(out), _ptr(a), a.nbytes,
                                     host_threads())
    if rc != SL_OK:
        raise SoftlatError(f"sl_host_copy failed ({rc})")
    return out


def masked_extrema(v: np.ndarray, mask: np.ndarray | None):
    """(min, max) of v where mask (threaded, sl_host_masked_extrema);
    numpy semantics: NaN propagates, empty gives (inf, -inf)."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    if mask is not None:
        mask = np.ascontiguousarray(mask).view(np.uint8)
        if len(mask) != len(v):
            raise InvalidValueError("mask length differs")
    lo, hi = C.c_double(), C.c_double()
    rc = load_library().sl_host_masked_extrema(
        _ptr(v), _ptr(mask), len(v), host_threads(), C.byref(lo), C.byref(hi))
    if rc != SL_OK:
        raise SoftlatError(f"sl_host_masked_extrema failed ({rc})")
    return lo.value, hi.value


def host_is_iota(ids: np.ndarray) -> bool:
    """ids == arange(len(ids)) (host threads)."""
    ids = np.ascontiguousarray(ids, np.int64)
    out = C.c_int(0)
    rc = load_library().sl_host_is_iota(_ptr(ids), len(ids), host_threads(),
                                        C.byref(out))
    if rc != SL_OK:
        raise SoftlatError(f"sl_host_is_iota failed ({rc})")
    return bool(out.value)


def host_copy_into(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[...] = src (same shape / dtype, contiguous) on the host threads."""
    src = np.ascontiguousarray(src)
    if dst.shape != src.shape or dst.dtype != src.dtype:
        raise InvalidValueError("host_copy_into: shape / dtype mismatch")
    if src.nbytes < (1 << 20):
        dst[...] = src
        return
    rc = load_library().sl_host_copy(_ptr(dst), _ptr(src), src.nbytes,
                                     host_threads())
    if rc != SL_OK:
        raise SoftlatError(f"sl_host_copy failed ({rc})")


def host_touch(a: np.ndarray) -> None:
    """First-touch every page of a fresh array (zero fill, host threads)."""
    zero = np.zeros(1, np.uint8)
    rc = load_library().sl_host_fill(_ptr(a), _ptr(zero), 1, a.nbytes,
                                     host_threads())
    if rc != SL_OK:
        raise SoftlatError(f"sl_host_fill failed ({rc})")


def is_pinned(a: np.ndarray) -> bool:
    base = a
    while True:
        if isinstance(base, np.ndarray) and base.base is not None:
            base = base.base
        elif isinstance(getattr(base, "_raw", None), np.ndarray):
            base = base._raw  # an owner object (control._Lease)
        else:
            break
    return isinstance(base, _PinnedBlock)


class Context:
    """One device context: SoA buffers of one store on one GPU + a stream."""

    def __init__(self, device: int = 0, precision: str = "fp64"):
        if precision not in PRECISIONS:
            raise InvalidValueError(
                f"precision must be one of {tuple(PRECISIONS)}")
        self.lib = load_library()
        self.device = int(device)
        self.precision = precision
        h = C.c_void_p()
        rc = self.lib.sl_create(self.device, PRECISIONS[precision],
                                C.byref(h))
        if rc != SL_OK:
            raise DeviceError(
                f"sl_create failed ({rc}): "
                f"{self.lib.sl_last_error(None).decode()}")
        self.h = h
        self.m_n = 0
        # advanced on every call that moves the device state past the host
        # copy (steps, single passes): the device mirror knows whether the
        # host store still equals the device after a pull
        self.epoch = 0
        self.s_n = 0

    # ------------------------------------------------------------ errors
    def _check(self, rc: int, what: str, mass_slot: int | None = None):
        if rc == SL_OK:
            return
        msg = self.lib.sl_last_error(self.h).decode()
        if rc == SL_ENUMERIC:
            raise NumericalAbort(
                f"non-finite state on mass slot {mass_slot}; reduce dt or "
                "stiffness", mass_slot=mass_slot)
        if rc == SL_EINVAL:
            raise InvalidValueError(f"{what}: {msg}")
        raise DeviceError(f"{what} failed ({rc}): {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.sl_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ upload
    def upload_masses(self, pos, vel, acc, fext, load, mass, fixed, alive,
                      gen):
        n = len(mass)
        a = [_c(pos, np.float64), _c(vel, np.float64), _c(acc, np.float64),
             _c(fext, np.float64), _c(load, np.float64),
             _c(mass, np.float64), _c(fixed, np.uint8), _c(alive, np.uint8),
             _c(gen, np.int64)]
        self._check(self.lib.sl_upload_masses(self.h, n, *map(_ptr, a)),
                    "sl_upload_masses")
        self.m_n = n

    def write_state(self, pos=None, vel=None, acc=None):
        """Whole pos / vel / acc columns into the context (sl_write_state);
        None keeps the device copy."""
        cols = [None if a is None else _c(a, np.float64)
                for a in (pos, vel, acc)]
        self._check(self.lib.sl_write_state(
            self.h, self.m_n, *[_ptr(a) if a is not None else None
                                for a in cols]), "sl_write_state")

    def write_state_async(self, pos=None, vel=None, acc=None):
        """sl_write_state_async: enqueued only; the arrays (contiguous fp64,
        page-locked) must stay unchanged until sync()."""
        for a in (pos, vel, acc):
            if a is not None and not (isinstance(a, np.ndarray) and
                                      a.dtype == np.float64 and
                                      a.flags.c_contiguous and
                                      a.size == 3 * self.m_n):
                raise InvalidValueError("write_state_async: pass contiguous "
                                        "float64 (m, 3) arrays")
        self._check(self.lib.sl_write_state_async(
            self.h, self.m_n, *[_ptr(a) if a is not None else None
                                for a in (pos, vel, acc)]),
            "sl_write_state_async")

    def upload_springs(self, m1, m2, m1gen, m2gen, rest, k, diam, yld, mode,
                       amp, freq, off, per, alive, degen):
        n = len(m1)
        a = [_c(m1, np.int64), _c(m2, np.int64), _c(m1gen, np.int64),
             _c(m2gen, np.int64), _c(rest, np.float64), _c(k, np.float64),
             _c(diam, np.float64), _c(yld, np.float64), _c(mode, np.int8),
             _c(amp, np.float64), _c(freq, np.float64), _c(off, np.float64),
             _c(per, np.float64), _c(alive, np.uint8), _c(degen, np.uint8)]
        self._check(self.lib.sl_upload_springs(self.h, n, *map(_ptr, a)),
                    "sl_upload_springs")
        self.s_n = n

    def set_environment(self, gravity, drag, planes, balls, gc_kind, gc_vec,
                        v_stick):
        g = _c(gravity, np.float64)
        pl = _c(np.reshape(planes, (-1, 7)), np.float64)
        bl = _c(np.reshape(balls, (-1, 5)), np.float64)
        gk = _c(gc_kind, np.int8)
        gv = _c(np.reshape(gc_vec, (-1, 3)), np.float64)
        self._check(self.lib.sl_set_environment(
            self.h, _ptr(g), float(drag), _ptr(pl), len(pl), _ptr(bl),
            len(bl), _ptr(gk), _ptr(gv), len(gk), float(v_stick)),
            "sl_set_environment")

    def set_local_constraints(self, lc_off, lc_kind, lc_vec):
        off = _c(lc_off, np.int64)
        kind = _c(lc_kind, np.int8)
        vec = _c(np.reshape(lc_vec, (-1, 3)), np.float64)
        self._check(self.lib.sl_set_local_constraints(
            self.h, len(off) - 1, _ptr(off), _ptr(kind), _ptr(vec),
            len(kind)), "sl_set_local_constraints")

    def set_custom_factors(self, slots, factors):
        s = _c(slots, np.int64)
        f = _c(factors, np.float64)
        self._check(self.lib.sl_set_custom_factors(self.h, len(s), _ptr(s),
                                                   _ptr(f)),
                    "sl_set_custom_factors")

    def write_masses(self, slots, pos, vel, acc, fext, load, mass, fixed,
                     alive, gen):
        s = _c(slots, np.int64)
        a = [_c(pos, np.float64), _c(vel, np.float64), _c(acc, np.float64),
             _c(fext, np.float64), _c(load, np.float64),
             _c(mass, np.float64), _c(fixed, np.uint8), _c(alive, np.uint8),
             _c(gen, np.int64)]
        self._check(self.lib.sl_write_masses(self.h, len(s), _ptr(s),
                                             *map(_ptr, a)),
                    "sl_write_masses")

    def write_spring_params(self, slots, rest, k, diam, yld, mode, amp, freq,
                            off, per):
        s = _c(slots, np.int64)
        a = [_c(rest, np.float64), _c(k, np.float64), _c(diam, np.float64),
             _c(yld, np.float64), _c(mode, np.int8), _c(amp, np.float64),
             _c(freq, np.float64), _c(off, np.float64), _c(per, np.float64)]
        self._check(self.lib.sl_write_spring_params(self.h, len(s), _ptr(s),
                                                    *map(_ptr, a)),
                    "sl_write_spring_params")

    def energy(self, sim_t: float, gravity) -> np.ndarray:
        """(kinetic, spring potential, gravitational potential)."""
        g = _c(gravity, np.float64)
        out = np.zeros(3)
        self._check(self.lib.sl_energy(self.h, float(sim_t), _ptr(g),
                                       _ptr(out)), "sl_energy")
        return out

    def spring_loads(self, sim_t: float, n: int):
        """(lengths, |F|) per spring slot [0, n); NaN for dead slots."""
        lengths, fmag = np.empty(n), np.empty(n)
        self._check(self.lib.sl_spring_loads(self.h, float(sim_t),
                                             _ptr(lengths), _ptr(fmag)),
                    "sl_spring_loads")
        return lengths, fmag

    def write_springs(self, slots, m1, m2, m1gen, m2gen, rest, k, diam, yld,
                      mode, amp, freq, off, per, alive, degen):
        s = _c(slots, np.int64)
        a = [_c(m1, np.int64), _c(m2, np.int64), _c(m1gen, np.int64),
             _c(m2gen, np.int64), _c(rest, np.float64), _c(k, np.float64),
             _c(diam, np.float64), _c(yld, np.float64), _c(mode, np.int8),
             _c(amp, np.float64), _c(freq, np.float64), _c(off, np.float64),
             _c(per, np.float64), _c(alive, np.uint8), _c(degen, np.uint8)]
        self._check(self.lib.sl_write_springs(self.h, len(s), _ptr(s),
                                              *map(_ptr, a)),
                    "sl_write_springs")

    def kill_springs(self, slots):
        s = _c(slots, np.int64)
        self._check(self.lib.sl_kill_springs(self.h, len(s), _ptr(s)),
                    "sl_kill_springs")

    # -------------------------------------------------------------- step
    def step(self, sim_times, dt: float, accumulation: int,
             counters: np.ndarray) -> tuple[int, int]:
        """Returns (steps_done, err_slot); raises NumericalAbort on a
        non-finite step (after the state of that step is resident)."""
        self.epoch += 1
        t = _c(sim_times, np.float64)
        err = C.c_int64(0)
        done = C.c_int64(0)
        rc = self.lib.sl_step(self.h, len(t), _ptr(t), float(dt),
                              int(accumulation), _ptr(counters),
                              C.byref(err), C.byref(done))
        if rc == SL_ENUMERIC:
            return int(done.value), int(err.value)
        self._check(rc, "sl_step")
        return int(done.value), 0

    def step_async(self, sim_times, dt: float, accumulation: int):
        """Enqueue steps without synchronising (sl_step_async)."""
        self.epoch += 1
        t = _c(sim_times, np.float64)
        self._check(self.lib.sl_step_async(self.h, len(t), _ptr(t),
                                           float(dt), int(accumulation)),
                    "sl_step_async")

    def step_finish(self, counters: np.ndarray) -> tuple[int, int]:
        """Synchronise an asynchronous run: (steps_done, err_slot)."""
        err = C.c_int64(0)
        done = C.c_int64(0)
        rc = self.lib.sl_step_finish(self.h, _ptr(counters), C.byref(err),
                                     C.byref(done))
        if rc == SL_ENUMERIC:
            return int(done.value), int(err.value)
        self._check(rc, "sl_step_finish")
        return int(done.value), 0

    def mark_ghosts(self, slots):
        s = _c(slots, np.int64)
        self._check(self.lib.sl_mark_ghosts(self.h, len(s), _ptr(s)),
                    "sl_mark_ghosts")

    def state_pointers(self) -> tuple[int, int, int]:
        """(device pointer of the position buffer the next step reads,
        rows, bytes per record)."""
        p = C.c_void_p()
        rows = C.c_int64(0)
        rb = C.c_int32(0)
        self._check(self.lib.sl_state_pointers(self.h, C.byref(p),
                                               C.byref(rows), C.byref(rb)),
                    "sl_state_pointers")
        return int(p.value or 0), int(rows.value), int(rb.value)

    def state_lo(self) -> int:
        """fp32 mode: device pointer of the position low parts of the
        buffer the next step reads (8 B per mass); 0 otherwise."""
        p = C.c_void_p()
        self._check(self.lib.sl_state_lo(self.h, C.byref(p)), "sl_state_lo")
        return int(p.value or 0)

    def stream(self) -> int:
        p = C.c_void_p()
        self._check(self.lib.sl_get_stream(self.h, C.byref(p)),
                    "sl_get_stream")
        return int(p.value or 0)

    def spring_pass(self, sim_t: float, accumulation: int,
                    counters: np.ndarray):
        self.epoch += 1
        self._check(self.lib.sl_spring_pass(self.h, float(sim_t),
                                            int(accumulation),
                                            _ptr(counters)),
                    "sl_spring_pass")

    def mass_pass(self, dt: float) -> int:
        self.epoch += 1
        err = C.c_int64(0)
        rc = self.lib.sl_mass_pass(self.h, float(dt), C.byref(err))
        if rc == SL_ENUMERIC:
            return int(err.value)
        self._check(rc, "sl_mass_pass")
        return 0

    # ----------------------------------------------------------- download
    def download_masses(self, pos=None, vel=None, acc=None, fext=None):
        for a in (pos, vel, acc, fext):
            if a is not None:
                assert a.dtype == np.float64 and a.flags.c_contiguous \
                    and a.shape == (self.m_n, 3)
        self._check(self.lib.sl_download_masses(
            self.h, _ptr(pos), _ptr(vel), _ptr(acc), _ptr(fext)),
            "sl_download_masses")

    def download_springs(self, alive=None, degen=None):
        for a in (alive, degen):
            if a is not None:
                assert a.itemsize == 1 and a.flags.c_contiguous \
                    and a.shape == (self.s_n,)
        self._check(self.lib.sl_download_springs(self.h, _ptr(alive),
                                                 _ptr(degen)),
                    "sl_download_springs")

    def snapshot_begin(self):
        self._check(self.lib.sl_snapshot_begin(self.h), "sl_snapshot_begin")

    def snapshot_ready(self) -> bool:
        r = C.c_int(0)
        self._check(self.lib.sl_snapshot_ready(self.h, C.byref(r)),
                    "sl_snapshot_ready")
        return bool(r.value)

    def snapshot_wait(self, pos=None, vel=None):
        self._check(self.lib.sl_snapshot_wait(self.h, _ptr(pos), _ptr(vel)),
                    "sl_snapshot_wait")

    # ------------------------------------------------------------- timing
    def timer_start(self):
        self._check(self.lib.sl_timer_start(self.h), "sl_timer_start")

    def timer_stop(self) -> float:
        ms = C.c_float(0.0)
        self._check(self.lib.sl_timer_stop(self.h, C.byref(ms)),
                    "sl_timer_stop")
        return float(ms.value)

    # ---------------------------------------------- in-library halo
    def halo_init(self, n_peers: int, dst: np.ndarray):
        """dst: int32 [m_n, 2], (row << 3) | peer or -1 (sl_halo_init)."""
        d = np.ascontiguousarray(dst, np.int32).reshape(-1)
        self._check(self.lib.sl_halo_init(self.h, int(n_peers), _ptr(d)),
                    "sl_halo_init")

    def halo_local(self) -> list[int]:
        p = (C.c_void_p * 5)()
        self._check(self.lib.sl_halo_local(self.h, p), "sl_halo_local")
        return [int(x or 0) for x in p]

    def halo_ipc_handles(self) -> bytes:
        buf = C.create_string_buffer(5 * 64)
        self._check(self.lib.sl_halo_ipc_handles(self.h, buf),
                    "sl_halo_ipc_handles")
        return buf.raw

    def halo_ipc_open(self, handles: bytes) -> list[int]:
        buf = C.create_string_buffer(bytes(handles), 5 * 64)
        p = (C.c_void_p * 5)()
        self._check(self.lib.sl_halo_ipc_open(self.h, buf, p),
                    "sl_halo_ipc_open")
        return [int(x or 0) for x in p]

    def halo_set_peer(self, peer: int, ptrs, slot: int):
        p = (C.c_void_p * 5)(*[x or None for x in ptrs])
        self._check(self.lib.sl_halo_set_peer(self.h, int(peer), p,
                                              int(slot)), "sl_halo_set_peer")

    def halo_commit(self):
        self._check(self.lib.sl_halo_commit(self.h), "sl_halo_commit")

    def set_spring_damping(self, damping):
        """Per-spring damping c for slots [0, s_n) (zeros clear it)."""
        d = _c(damping, np.float64)
        self._check(self.lib.sl_set_spring_damping(self.h, len(d), _ptr(d)),
                    "sl_set_spring_damping")

    def download_state(self, pos, vel, acc, fext):
        """pos / vel now; acc / f_ext (page-locked) land asynchronously --
        download_wait() before reading them."""
        self._check(self.lib.sl_download_state(
            self.h, *[_ptr(a) if a is not None else None
                      for a in (pos, vel, acc, fext)]), "sl_download_state")

    def download_state_ex(self, pos, vel, acc, fext, pos2=None, vel2=None,
                          wait_head=False):
        """sl_download_state_ex: every destination page-locked and kept
        alive by the caller until download_wait() (pos2 / vel2:
        download_wait_extra())."""
        for a in (pos, vel, acc, fext, pos2, vel2):
            if a is not None and not (a.dtype == np.float64 and
                                      a.flags.c_contiguous and
                                      a.size == 3 * self.m_n):
                raise InvalidValueError("download_state_ex: contiguous "
                                        "float64 (m, 3) arrays")
        self._check(self.lib.sl_download_state_ex(
            self.h, *[_ptr(a) if a is not None else None
                      for a in (pos, vel, acc, fext, pos2, vel2)],
            1 if wait_head else 0), "sl_download_state_ex")

    def stash_state(self):
        self._check(self.lib.sl_stash_state(self.h), "sl_stash_state")

    def download_stash(self, pos=None, vel=None, acc=None, fext=None):
        """Stashed state (sl_stash_state) into host arrays; waits."""
        for a in (pos, vel, acc, fext):
            if a is not None and not (a.dtype == np.float64 and
                                      a.flags.c_contiguous and
                                      a.size == 3 * self.m_n):
                raise InvalidValueError("download_stash: contiguous "
                                        "float64 (m, 3) arrays")
        self._check(self.lib.sl_download_stash(
            self.h, *[_ptr(a) if a is not None else None
                      for a in (pos, vel, acc, fext)]), "sl_download_stash")

    def checkpoint(self, view_pos=None, view_vel=None):
        """sl_checkpoint (views: page-locked (m, 3) fp64, kept alive until
        checkpoint_view_wait())."""
        for a in (view_pos, view_vel):
            if a is not None and not (a.dtype == np.float64 and
                                      a.flags.c_contiguous and
                                      a.size == 3 * self.m_n):
                raise InvalidValueError("checkpoint: contiguous float64 "
                                        "(m, 3) arrays")
        self._check(self.lib.sl_checkpoint(
            self.h, *[_ptr(a) if a is not None else None
                      for a in (view_pos, view_vel)]), "sl_checkpoint")

    def checkpoint_view_wait(self):
        self._check(self.lib.sl_checkpoint_view_wait(self.h),
                    "sl_checkpoint_view_wait")

    def restore(self):
        self.epoch += 1
        self._check(self.lib.sl_restore(self.h), "sl_restore")

    def download_wait_extra(self):
        self._check(self.lib.sl_download_wait_extra(self.h),
                    "sl_download_wait_extra")

    def download_wait(self):
        self._check(self.lib.sl_download_wait(self.h), "sl_download_wait")

    def last_step_ms(self) -> float:
        """Device time of the step kernels of the last step() call."""
        ms = C.c_float(0.0)
        self._check(self.lib.sl_last_step_ms(self.h, C.byref(ms)),
                    "sl_last_step_ms")
        return float(ms.value)

    def sync(self):
        self._check(self.lib.sl_sync(self.h), "sl_sync")

    def stats(self) -> dict:
        st = SlStats()
        self._check(self.lib.sl_get_stats(self.h, C.byref(st)),
                    "sl_get_stats")
        return {f: getattr(st, f) for f, _ in SlStats._fields_}
