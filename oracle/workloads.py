"""Bench workloads as oracle cases, built with numpy only.

TEST INFRASTRUCTURE (like the rest of oracle/): the reference arm of
bench.py (``--impl reference``) and its CPU baseline leg build their inputs
here, so the reference run maps nothing from the product package -- no
``paper_1911_10274_b200`` import, no libsoftlat_cuda.so.  The arrays are
the reference builder's, restated:

* lattice enumeration -- row-major node ids ``(i*ny + j)*nz + k``, the 13
  same-cell offsets in the reference order, springs grouped by offset, each
  group in row-major order of its lower node
  (/root/reference/pkg/src/softlat/builder.py:28-30, 112-138);
* materialisation -- rest length = build-time distance
  ``sqrt((dx*dx + dy*dy) + dz*dz)``, k = E*A/L with A = pi (d/2)^2, node
  mass = sum of half-bar masses in ``np.add.at`` order (builder.py:141-174);
* the bench recipe -- spacing 0.05, E = 1e5, rho = 1000, positions x1.01
  (cli.py:263-271); config A = scenarios/bouncing_cube.ini;
* robot swarms stacked along +y with a two-spacing gap (cli.py:323-331),
  worm actuation offsets ``min(x_a, x_b) - min x`` (actuation.py:72-111;
  t_p = 1, omega = 20, c = 0.2: actuation.py:22-25).

tests/test_workloads.py checks these cases equal the product builder's
stores array for array (the product builder is itself pinned to the
reference's goldens, tests/test_builder.py).
"""
from __future__ import annotations

import math

import numpy as np

CELL_OFFSETS = ((1, 0, 0), (0, 1, 0), (0, 0, 1),
                (1, 1, 0), (1, -1, 0), (1, 0, 1), (1, 0, -1),
                (0, 1, 1), (0, 1, -1),
                (1, 1, 1), (1, 1, -1), (1, -1, 1), (1, -1, -1))
MIN_NODE_MASS = 1e-9
ACT_SINE = 1
WORM = dict(amplitude=0.2, frequency=20.0, period=1.0)


def grid_springs(nx, ny, nz):
    a_parts, b_parts = [], []
    for dx, dy, dz in CELL_OFFSETS:
        lo = (max(0, -dx), max(0, -dy), max(0, -dz))
        hi = (nx - max(0, dx), ny - max(0, dy), nz - max(0, dz))
        if any(h <= l for l, h in zip(lo, hi)):
            continue
        ii = np.arange(lo[0], hi[0])[:, None, None]
        jj = np.arange(lo[1], hi[1])[None, :, None]
        kk = np.arange(lo[2], hi[2])[None, None, :]
        a_parts.append(((ii * ny + jj) * nz + kk).reshape(-1))
        b_parts.append((((ii + dx) * ny + (jj + dy)) * nz + (kk + dz))
                       .reshape(-1))
    if not a_parts:
        z = np.zeros(0, np.int64)
        return z, z.copy()
    return (np.concatenate(a_parts).astype(np.int64),
            np.concatenate(b_parts).astype(np.int64))


def grid_positions(corner, nx, ny, nz, spacing):
    idx = np.indices((nx, ny, nz)).reshape(3, -1).T
    return np.asarray(corner, np.float64) + spacing * idx.astype(np.float64)


def materialize(pos, a, b, E, rho, diameter):
    d = pos[b] - pos[a]
    rest = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])
    diam = np.full(rest.shape, float(diameter))
    area = math.pi * (diam * 0.5) ** 2
    stiff = E * area / rest
    half = 0.5 * rho * area * rest
    mass = np.zeros(len(pos))
    np.add.at(mass, a, half)
    np.add.at(mass, b, half)
    mass[mass <= 0.0] = MIN_NODE_MASS
    return rest, stiff, diam, mass


def make_case(pos, mass, a, b, rest, stiff, diam, gravity, planes,
              drag=0.0):
    m, s = len(pos), len(a)
    z3 = np.zeros((m, 3))
    return {
        "m_pos": np.ascontiguousarray(pos, np.float64), "m_vel": z3.copy(),
        "m_acc": z3.copy(), "m_fext": z3.copy(), "m_load": z3.copy(),
        "m_mass": mass, "m_fixed": np.zeros(m, np.uint8),
        "m_alive": np.ones(m, np.uint8), "m_gen": np.zeros(m, np.int64),
        "s_m1": a, "s_m2": b, "s_m1gen": np.zeros(s, np.int64),
        "s_m2gen": np.zeros(s, np.int64), "s_rest": rest, "s_k": stiff,
        "s_diam": diam, "s_yield": np.full(s, np.inf),
        "s_mode": np.zeros(s, np.int8), "s_amp": np.zeros(s),
        "s_freq": np.zeros(s), "s_off": np.zeros(s), "s_per": np.ones(s),
        "s_alive": np.ones(s, np.uint8), "s_degen": np.zeros(s, np.uint8),
        "gravity": np.asarray(gravity, np.float64), "drag": float(drag),
        "planes": np.asarray(planes, np.float64).reshape(-1, 7),
        "balls": np.zeros((0, 5)), "gc_kind": np.zeros(0, np.int8),
        "gc_vec": np.zeros((0, 3)), "lc_off": np.zeros(m + 1, np.int64),
        "lc_kind": np.zeros(0, np.int8), "lc_vec": np.zeros((0, 3)),
    }


def ground(k, mu_s=1.0, mu_k=0.8):
    """ContactPlane(normal +z, offset 0) flattened as engine.py:223-236."""
    return np.array([[0.0, 0.0, 1.0, 0.0, k, mu_s, mu_k]])


def config_b(n=100):
    """n^3 bench lattice, x1.01 stretch, gravity, friction ground plane
    (k 2000, mu_s 1, mu_k 0.8) with the bottom layer on it."""
    pos = grid_positions((0.0, 0.0, 0.0), n, n, n, 0.05)
    a, b = grid_springs(n, n, n)
    rest, stiff, diam, mass = materialize(pos, a, b, 1e5, 1000.0, 1e-3)
    pos = pos * 1.01
    return make_case(pos, mass, a, b, rest, stiff, diam, (0, 0, -9.81),
                     ground(2000.0))


def config_a():
    """scenarios/bouncing_cube.ini: 10^3 lattice at (0, 0, 0.3), spacing
    0.1, E 1e6, rho 1000, d 1 mm, ground k 2000."""
    pos = grid_positions((0.0, 0.0, 0.3), 10, 10, 10, 0.1)
    a, b = grid_springs(10, 10, 10)
    rest, stiff, diam, mass = materialize(pos, a, b, 1e6, 1000.0, 1e-3)
    return make_case(pos, mass, a, b, rest, stiff, diam, (0, 0, -9.81),
                     ground(2000.0))


def config_d(count=4096, first=0, edge=5):
    """``count`` worm-actuated edge^3 robots (spacing 0.05, E 1e6) stacked
    along +y, robots first.. of the global swarm; ground k 500, drag
    0.01."""
    sp = 0.05
    pos1 = grid_positions((0.0, 0.0, 0.0), edge, edge, edge, sp)
    a1, b1 = grid_springs(edge, edge, edge)
    step = (edge - 1) * sp + 2 * sp
    shift = np.zeros((count, 1, 3))
    shift[:, 0, 1] = (first + np.arange(count)) * step
    pos = (pos1[None] + shift).reshape(-1, 3)
    base = (np.arange(count) * len(pos1))[:, None]
    a = (a1[None] + base).reshape(-1)
    b = (b1[None] + base).reshape(-1)
    rest, stiff, diam, mass = materialize(pos, a, b, 1e6, 1000.0, 1e-3)
    case = make_case(pos, mass, a, b, rest, stiff, diam, (0, 0, -9.81),
                     ground(500.0), drag=0.01)
    x0 = pos1[:, 0]
    off1 = np.minimum(x0[a1], x0[b1]) - x0.min()
    case["s_mode"][:] = ACT_SINE
    case["s_amp"][:] = WORM["amplitude"]
    case["s_freq"][:] = WORM["frequency"]
    case["s_off"][:] = np.tile(off1, count)
    case["s_per"][:] = WORM["period"]
    return case


def workload(config: str, n: int = 100, robots: int = 4096):
    if config == "A":
        return config_a()
    if config == "D":
        return config_d(robots)
    return config_b(n)
