"""Snapshot, energy-log and report files (the reference's io.py).

Same formats and names as io.py:1-80.  ``format_snapshot`` /
``write_snapshot`` produce byte-identical text (Python's ``{:.17g}`` digits,
io.py:19-27) through the library's threaded formatter
(``sl_format_snapshot``, csrc/sl_host.cpp) instead of a per-row Python loop;
``read_snapshot`` parses with numpy's C reader and falls back to the
reference's line loop for its error messages (io.py:35-49).  Binary
snapshots (``write_snapshot_npz`` / ``read_snapshot_npz``) are the
lossless fast format SURVEY.md 8(f) rank 4 asks for beside the CSV.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from pathlib import Path

import numpy as np

from . import _native
from .errors import ScenarioError
from .store import ObjectStore

SNAPSHOT_HEADER = "id,x,y,z,vx,vy,vz"


def _threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def format_snapshot_bytes(ids: np.ndarray, positions: np.ndarray,
                          velocities: np.ndarray) -> memoryview:
    """The snapshot text (io.py:19-27) as ASCII bytes."""
    ids = np.ascontiguousarray(ids, dtype=np.int64).reshape(-1)
    pos = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
    vel = np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3)
    n = len(ids)
    if len(pos) != n or len(vel) != n:
        raise ValueError("ids, positions and velocities differ in length")
    cap = len(SNAPSHOT_HEADER) + 1 + n * _native_row_max()
    out = np.empty(cap, np.uint8)
    used = C.c_size_t(0)
    lib = _native.load_library()
    rc = lib.sl_format_snapshot(n, _native._ptr(ids), _native._ptr(pos),
                                _native._ptr(vel), _threads(),
                                _native._ptr(out), cap, C.byref(used))
    if rc != _native.SL_OK:
        raise ValueError(f"sl_format_snapshot failed ({rc})")
    return memoryview(out[:used.value])


def _native_row_max() -> int:
    return 176  # SL_SNAPSHOT_ROW_MAX, include/softlat_cuda.h


def format_snapshot(ids: np.ndarray, positions: np.ndarray,
                    velocities: np.ndarray) -> str:
    return bytes(format_snapshot_bytes(ids, positions, velocities)).decode(
        "ascii")


def write_snapshot(path, ids: np.ndarray, positions: np.ndarray,
                   velocities: np.ndarray) -> None:
    data = format_snapshot_bytes(ids, positions, velocities)
    with open(path, "wb") as fh:
        fh.write(data)


def _read_snapshot_lines(path, lines):
    """io.py:35-49, line for line (errors and messages)."""
    ids, pos, vel = [], [], []
    for ln, line in enumerate(lines[1:], start=2):
        parts = line.split(",")
        if len(parts) != 7:
            raise ScenarioError(f"{path}:{ln}: expected 7 columns")
        ids.append(int(parts[0]))
        vals = [float(p) for p in parts[1:]]
        pos.append(vals[:3])
        vel.append(vals[3:])
    return (np.array(ids, dtype=np.int64),
            np.array(pos).reshape(-1, 3), np.array(vel).reshape(-1, 3))


def read_snapshot(path) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    lines = Path(path).read_text().strip().splitlines()
    if not lines or lines[0].strip() != SNAPSHOT_HEADER:
        raise ScenarioError(f"{path}: not a snapshot file (bad header)")
    data = lines[1:]
    if not data:
        return (np.zeros(0, np.int64), np.zeros((0, 3)), np.zeros((0, 3)))
    try:
        # numpy's C parser (correctly rounded, like float()); anything it
        # skips or reads differently from the reference's loop (blank lines,
        # other column counts) goes to that loop instead
        ids = np.loadtxt(data, delimiter=",", usecols=0, dtype=np.int64,
                         ndmin=1, comments=None)
        vals = np.loadtxt(data, delimiter=",", usecols=range(1, 7),
                          dtype=np.float64, ndmin=2, comments=None)
        if vals.shape != (len(data), 6) or len(ids) != len(data) or \
                sum(ln.count(",") for ln in data) != 6 * len(data):
            raise ValueError("column count")
        return ids, vals[:, :3].copy(), vals[:, 3:].copy()
    except ValueError:
        return _read_snapshot_lines(path, lines)


def apply_snapshot(store: ObjectStore, ids: np.ndarray, positions: np.ndarray,
                   velocities: np.ndarray) -> None:
    """Overwrite positions/velocities of the given alive slots (io.py:52-59)."""
    n = store.mass_slot_count
    ids = np.asarray(ids)
    from . import _native
    pos = np.ascontiguousarray(positions, np.float64)
    vel = np.ascontiguousarray(velocities, np.float64)
    if len(ids) == n and store.mass_count == n and len(ids) and \
            ids[0] == 0 and ids[-1] == n - 1 and pos.size == 3 * n and \
            vel.size == 3 * n:
        # every slot, in order (checked below, while the upload runs):
        # whole-column copies (threaded, into the page-locked store
        # columns); a device mirror holding the rest of the state receives
        # the same columns meanwhile, straight from page-locked inputs
        # (engine.write_through_begin)
        from . import engine
        pos = pos.reshape(n, 3)
        vel = vel.reshape(n, 3)
        started = engine.write_through_begin(store, pos, vel)
        if not _native.host_is_iota(ids):  # not every slot in order
            engine.write_through_abort(store, started)
            return _apply_rows(store, ids, positions, velocities)
        # every device copy took the columns: the store's own copy is
        # deferred (filled from the device on first host need) instead of
        # paying a host memory copy now
        copy = not engine.write_through_covers(store, started)
        try:
            if copy:
                dst_pos, dst_vel = store._overwrite_state_columns()
                _native.host_copy_into(dst_pos[:n], pos)
                _native.host_copy_into(dst_vel[:n], vel)
        finally:
            engine.write_through_end(store, started, host_copied=copy)
        return
    _apply_rows(store, ids, positions, velocities)


def _apply_rows(store: ObjectStore, ids, positions, velocities) -> None:
    n = store.mass_slot_count
    if np.any(ids < 0) or np.any(ids >= n) or not np.all(store._m_alive[ids]):
        raise ScenarioError("snapshot ids do not match alive store slots")
    store._m_pos[ids] = positions
    store._m_vel[ids] = velocities


def write_snapshot_npz(path, ids: np.ndarray, positions: np.ndarray,
                       velocities: np.ndarray) -> None:
    """Binary snapshot: the same three arrays, lossless, no text."""
    with open(path, "wb") as fh:
        np.savez(fh, ids=np.asarray(ids, np.int64),
                 positions=np.asarray(positions, np.float64).reshape(-1, 3),
                 velocities=np.asarray(velocities, np.float64).reshape(-1, 3))


def read_snapshot_npz(path) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    try:
        with np.load(path) as z:
            return z["ids"], z["positions"], z["velocities"]
    except (OSError, KeyError, ValueError) as exc:
        raise ScenarioError(f"{path}: not a binary snapshot ({exc})") from exc


class EnergyLog:
    """Per-snapshot energy rows written as CSV (io.py:62-80)."""

    HEADER = "sim_time,kinetic,spring_potential,gravity_potential,total"

    def __init__(self):
        self.rows: list[tuple[float, float, float, float]] = []

    def add(self, sim_time: float, energy) -> None:
        self.rows.append((sim_time, energy.kinetic, energy.spring_potential,
                          energy.gravity_potential))

    def write(self, path) -> None:
        lines = [self.HEADER]
        for t, ke, spe, gpe in self.rows:
            lines.append(f"{t:.17g},{ke:.17g},{spe:.17g},{gpe:.17g},"
                         f"{ke + spe + gpe:.17g}")
        Path(path).write_text("\n".join(lines) + "\n")


def write_report(path, report: dict) -> None:
    Path(path).write_text(json.dumps(report, indent=2, default=str) + "\n")
