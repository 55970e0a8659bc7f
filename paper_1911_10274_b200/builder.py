"""Lattice construction (host side; generates every synthetic input).

Reproduces the reference builder's enumeration bit for bit
(/root/reference/pkg/src/softlat/builder.py:112-186): row-major node ids
``(i*ny + j)*nz + k``, the 13 canonical same-cell offsets in the reference
order, springs grouped by offset, rest length = exact build-time endpoint
distance, k = E*A/L (bar model), node mass = sum of half-bar masses.  Slot
order fixes the per-mass accumulation order on the device, so "connectivity
and indexing bit-exact" (north_star) starts here; tests/test_builder.py
checks these arrays against the reference-generated golden inputs.

STL / mesh fills are out of scope (component 8).
"""
from __future__ import annotations

import logging
import math
from dataclasses import dataclass, field

import numpy as np

from .core import Material, Vec3
from .errors import InvalidValueError
from .store import HandleBatch, ObjectStore

log = logging.getLogger(__name__)

MIN_NODE_MASS = 1e-9

# 3 axis, 6 face-diagonal, 4 body-diagonal offsets (builder.py:28-30 order)
CELL_OFFSETS = ((1, 0, 0), (0, 1, 0), (0, 0, 1),
                (1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1),
                (0, 1, 1), (0, 1, -1),
                (1, 1, 1), (1, 1, -1), (1, -1, 1), (1, -1, -1))


@dataclass(frozen=True)
class LatticeSpec:
    corner: Vec3
    nx: int
    ny: int
    nz: int
    spacing: float
    material: Material
    diameter: float = 1e-3

    def __post_init__(self):
        if min(self.nx, self.ny, self.nz) < 1:
            raise InvalidValueError("lattice counts must be >= 1")
        if self.spacing <= 0:
            raise InvalidValueError("lattice spacing must be positive")
        if self.diameter < 0:
            raise InvalidValueError("spring diameter must be >= 0")


@dataclass
class BodyHandle:
    """Handles of one built body plus its build-time geometry."""

    mass_handles: HandleBatch
    spring_handles: HandleBatch
    initial_positions: np.ndarray
    grid_indices: np.ndarray | None = None

    def center_of_mass(self, store: ObjectStore) -> Vec3:
        slots = self.mass_handles.slots
        s = slots[store._m_alive[slots]]
        if len(s) == 0:
            raise InvalidValueError("body has no alive masses")
        m = store._m_mass[s]
        return Vec3.of((store._m_pos[s] * m[:, None]).sum(axis=0) / m.sum())

    def mass_slots_where(self, predicate) -> np.ndarray:
        if self.grid_indices is None:
            raise InvalidValueError("body has no grid indices")
        return self.mass_handles.slots[predicate(self.grid_indices)]


@dataclass
class CubeGridBody(BodyHandle):
    """grid_x * grid_y cubes bridged by thin connector springs."""

    cube_members: list = field(default_factory=list)
    connector_rows: np.ndarray | None = None

    def cube_center_of_mass(self, store: ObjectStore, cube: int) -> Vec3:
        slots = self.mass_handles.slots[self.cube_members[cube]]
        s = slots[store._m_alive[slots]]
        m = store._m_mass[s]
        return Vec3.of((store._m_pos[s] * m[:, None]).sum(axis=0) / m.sum())


def derive_spring_constant(material: Material, diameter: float,
                           rest_length: float) -> float:
    if rest_length <= 0:
        raise InvalidValueError("rest length must be positive")
    if diameter < 0:
        raise InvalidValueError("diameter must be >= 0")
    return material.elastic_modulus * (math.pi * (diameter * 0.5) ** 2) \
        / rest_length


def derive_mass(material: Material, bars) -> float:
    total = 0.0
    for length, diameter in bars:
        total += 0.5 * material.density * (math.pi * (diameter * 0.5) ** 2) \
            * length
    if total <= 0.0:
        log.warning("node has no bar volume; assigning minimum mass %g kg",
                    MIN_NODE_MASS)
        return MIN_NODE_MASS
    return total


def lattice_spring_count(nx: int, ny: int, nz: int) -> int:
    ex, ey, ez = nx - 1, ny - 1, nz - 1
    return (ny * nz * ex + nx * nz * ey + nx * ny * ez
            + 2 * (nz * ex * ey + ny * ex * ez + nx * ey * ez)
            + 4 * ex * ey * ez)


def grid_springs(nx: int, ny: int, nz: int):
    """(a_ids, b_ids): every same-cell node pair, grouped by offset in
    CELL_OFFSETS order, each group in row-major order of its lower node."""
    a_parts, b_parts = [], []
    for dx, dy, dz in CELL_OFFSETS:
        lo = (max(0, -dx), max(0, -dy), max(0, -dz))
        hi = (nx - max(0, dx), ny - max(0, dy), nz - max(0, dz))
        if any(h <= l for l, h in zip(lo, hi)):
            continue
        ii = np.arange(lo[0], hi[0])[:, None, None]
        jj = np.arange(lo[1], hi[1])[None, :, None]
        kk = np.arange(lo[2], hi[2])[None, None, :]
        a = (ii * ny + jj) * nz + kk
        b = ((ii + dx) * ny + (jj + dy)) * nz + (kk + dz)
        a_parts.append(a.reshape(-1))
        b_parts.append(b.reshape(-1))
    if not a_parts:
        z = np.zeros(0, dtype=np.int64)
        return z, z.copy()
    return (np.concatenate(a_parts).astype(np.int64),
            np.concatenate(b_parts).astype(np.int64))


def _grid_positions(corner: Vec3, nx, ny, nz, spacing):
    idx = np.indices((nx, ny, nz)).reshape(3, -1).T
    return corner.as_array() + spacing * idx.astype(np.float64), idx


def materialize(store: ObjectStore, positions: np.ndarray, a_ids, b_ids,
                material: Material, diameter, fixed=None,
                grid_indices=None) -> BodyHandle:
    """Create masses + springs; rest length is the exact build-time distance
    computed with the kernel's expression ((dx*dx + dy*dy) + dz*dz)."""
    d = positions[b_ids] - positions[a_ids]
    rests = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])
    if np.any(rests <= 0):
        raise InvalidValueError("coincident lattice nodes")
    diam = np.broadcast_to(np.asarray(diameter, np.float64), rests.shape)
    area = math.pi * (diam * 0.5) ** 2
    stiff = material.elastic_modulus * area / rests
    half_bar = 0.5 * material.density * area * rests
    node_mass = np.zeros(len(positions))
    np.add.at(node_mass, a_ids, half_bar)
    np.add.at(node_mass, b_ids, half_bar)
    return _create(store, positions, node_mass, a_ids, b_ids, rests, stiff,
                   diam, material, fixed, grid_indices)


def _create(store, positions, node_mass, a_ids, b_ids, rests, stiff, diam,
            material, fixed, grid_indices) -> BodyHandle:
    bare = node_mass <= 0.0
    if bare.any():
        log.warning("%d nodes have no bar volume; assigning minimum mass %g kg",
                    int(bare.sum()), MIN_NODE_MASS)
        node_mass[bare] = MIN_NODE_MASS
    mh = store.create_masses(positions, node_mass, fixed=fixed)
    sh = store.create_springs(mh.slots[a_ids], mh.slots[b_ids], rests, stiff,
                              diameters=diam,
                              yield_stress=material.yield_stress)
    return BodyHandle(mass_handles=mh, spring_handles=sh,
                      initial_positions=positions.copy(),
                      grid_indices=grid_indices)


def _threads() -> int:
    import os
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def lattice_arrays(spec: LatticeSpec):
    """(positions, node_mass, a, b, rest, stiff) of ``spec`` from the
    library's threaded generator (sl_build_lattice), bit-identical to
    ``_grid_positions`` + ``grid_springs`` + ``materialize``'s numpy."""
    import ctypes as C
    from . import _native
    lib = _native.load_library()
    nm, ns = C.c_int64(), C.c_int64()
    if lib.sl_lattice_counts(spec.nx, spec.ny, spec.nz, C.byref(nm),
                             C.byref(ns)) != _native.SL_OK:
        raise InvalidValueError("bad lattice counts")
    nm, ns = nm.value, ns.value
    pos = np.empty((nm, 3))
    node_mass = np.empty(nm)
    a = np.empty(ns, np.int64)
    b = np.empty(ns, np.int64)
    rest = np.empty(ns)
    stiff = np.empty(ns)
    corner = spec.corner.as_array()
    m = spec.material
    p = _native._ptr
    rc = lib.sl_build_lattice(spec.nx, spec.ny, spec.nz, p(corner),
                              float(spec.spacing), float(m.elastic_modulus),
                              float(m.density), float(spec.diameter),
                              _threads(), p(pos), p(node_mass), p(a), p(b),
                              p(rest), p(stiff))
    if rc != _native.SL_OK:
        raise InvalidValueError(f"sl_build_lattice failed ({rc})")
    return pos, node_mass, a, b, rest, stiff


def build_lattice(spec: LatticeSpec, store: ObjectStore) -> BodyHandle:
    """builder.py:112-186: generated by the library (threads), same arrays
    as the numpy path (``build_lattice_numpy``, tests/test_builder.py)."""
    pos, node_mass, a, b, rest, stiff = lattice_arrays(spec)
    if not np.all(np.isfinite(pos)):
        raise InvalidValueError("non-finite mass position")
    if len(rest) and not np.all(rest > 0):
        raise InvalidValueError("coincident lattice nodes")
    idx = np.indices((spec.nx, spec.ny, spec.nz)).reshape(3, -1).T
    diam = np.broadcast_to(np.asarray(spec.diameter, np.float64), rest.shape)
    return _create(store, pos, node_mass, a, b, rest, stiff, diam,
                   spec.material, None, idx)


def build_lattice_numpy(spec: LatticeSpec, store: ObjectStore) -> BodyHandle:
    positions, idx = _grid_positions(spec.corner, spec.nx, spec.ny, spec.nz,
                                     spec.spacing)
    a, b = grid_springs(spec.nx, spec.ny, spec.nz)
    return materialize(store, positions, a, b, spec.material, spec.diameter,
                       grid_indices=idx)


def build_swarm(spec: LatticeSpec, store: ObjectStore, count: int,
                gap: float | None = None) -> list[BodyHandle]:
    """``count`` copies of a lattice stacked along +y with a two-spacing gap
    (the layout of cmd_swarm, cli.py:323-331).  Bodies are disjoint
    connected components in contiguous slot ranges -- the natural shard."""
    extent = (spec.ny - 1) * spec.spacing
    step = extent + 2 * spec.spacing if gap is None else extent + gap
    bodies = []
    for i in range(count):
        corner = Vec3(spec.corner.x, spec.corner.y + i * step, spec.corner.z)
        bodies.append(build_lattice(
            LatticeSpec(corner, spec.nx, spec.ny, spec.nz, spec.spacing,
                        spec.material, spec.diameter), store))
    return bodies


def build_robot_swarm(spec: LatticeSpec, store: ObjectStore, count: int,
                      worm: bool = True, gap: float | None = None,
                      first: int = 0):
    """``count`` lattice robots stacked along +y (cmd_swarm layout,
    cli.py:323-331) created in ONE bulk call, each worm-actuated like
    ``configure_worm`` (actuation.py:72-111) when ``worm``.  Same arrays as
    ``build_swarm`` + per-body ``configure_worm``, built vectorised (config
    D: thousands of RL robots).  ``first`` places the robots as robots
    first.. of a larger swarm (a rank's shard).  Returns per-body (mass
    slot range, spring slot range)."""
    from .actuation import WORM_AMPLITUDE, WORM_FREQUENCY, WORM_PERIOD
    pos1, idx = _grid_positions(spec.corner, spec.nx, spec.ny, spec.nz,
                                spec.spacing)
    a1, b1 = grid_springs(spec.nx, spec.ny, spec.nz)
    extent = (spec.ny - 1) * spec.spacing
    step = extent + 2 * spec.spacing if gap is None else extent + gap
    m1, s1 = len(pos1), len(a1)
    shift = np.zeros((count, 1, 3))
    # robot i of the global swarm sits at i * step; ``first`` makes a shard
    # (robots first .. first+count-1) bit-identical to that part of it
    shift[:, 0, 1] = (first + np.arange(count)) * step
    positions = (pos1[None] + shift).reshape(-1, 3)
    base = (np.arange(count) * m1)[:, None]
    a = (a1[None] + base).reshape(-1)
    b = (b1[None] + base).reshape(-1)
    body = materialize(store, positions, a, b, spec.material, spec.diameter)
    if worm:
        x0 = pos1[:, 0]
        off1 = np.minimum(x0[a1], x0[b1]) - x0.min()
        store.set_actuation_bulk(body.spring_handles.slots, WORM_AMPLITUDE,
                                 WORM_FREQUENCY, np.tile(off1, count),
                                 WORM_PERIOD)
    ms, ss = body.mass_handles.slots, body.spring_handles.slots
    return [((int(ms[i * m1]), int(ms[i * m1]) + m1),
             (int(ss[i * s1]), int(ss[i * s1]) + s1)) for i in range(count)]


def build_cube_grid(grid_x: int, grid_y: int, cube_counts, spacing: float,
                    material: Material, store: ObjectStore,
                    corner: Vec3 = Vec3(0, 0, 0), diameter: float = 1e-3,
                    connector_diameter: float = 4e-4) -> CubeGridBody:
    """Multi-body assembly joined along top/bottom layers
    (builder.py:206-265)."""
    if grid_x < 1 or grid_y < 1:
        raise InvalidValueError("cube grid counts must be >= 1")
    cx, cy, cz = cube_counts
    per = cx * cy * cz
    local = np.indices((cx, cy, cz)).reshape(3, -1).T.astype(np.float64)
    base = Vec3.of(corner).as_array()
    pos_parts, members = [], []
    for gi in range(grid_x):
        for gj in range(grid_y):
            origin = base + spacing * np.array([gi * cx, gj * cy, 0],
                                               dtype=np.float64)
            pos_parts.append(origin + spacing * local)
            start = (gi * grid_y + gj) * per
            members.append(np.arange(start, start + per))
    positions = np.vstack(pos_parts)

    def node(gi, gj, i, j, k):
        return (gi * grid_y + gj) * per + (i * cy + j) * cz + k

    la, lb = grid_springs(cx, cy, cz)
    n_cubes = grid_x * grid_y
    a_parts = [la + c * per for c in range(n_cubes)]
    b_parts = [lb + c * per for c in range(n_cubes)]
    diam_parts = [np.full(len(la) * n_cubes, diameter)]
    ca, cb = [], []
    for gi in range(grid_x):
        for gj in range(grid_y):
            for k in (0, cz - 1):
                if gi + 1 < grid_x:
                    for j in range(cy):
                        ca.append(node(gi, gj, cx - 1, j, k))
                        cb.append(node(gi + 1, gj, 0, j, k))
                if gj + 1 < grid_y:
                    for i in range(cx):
                        ca.append(node(gi, gj, i, cy - 1, k))
                        cb.append(node(gi, gj + 1, i, 0, k))
    n_internal = len(la) * n_cubes
    if ca:
        a_parts.append(np.array(ca, dtype=np.int64))
        b_parts.append(np.array(cb, dtype=np.int64))
        diam_parts.append(np.full(len(ca), connector_diameter))
    body = materialize(store, positions, np.concatenate(a_parts),
                       np.concatenate(b_parts), material,
                       np.concatenate(diam_parts))
    return CubeGridBody(mass_handles=body.mass_handles,
                        spring_handles=body.spring_handles,
                        initial_positions=body.initial_positions,
                        cube_members=members,
                        connector_rows=np.arange(n_internal,
                                                 len(body.spring_handles)))
