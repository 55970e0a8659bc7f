"""Snapshot writer throughput: the native threaded formatter vs the
reference's per-row loop (io.py:19-27, restated), 1M rows of config-B-like
state; binary (npz) for comparison."""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_10274_b200 import io as sio  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)
ids = np.arange(n, dtype=np.int64)
pos = rng.uniform(0, 5, (n, 3))
vel = rng.normal(0, 1e-2, (n, 3))
with tempfile.TemporaryDirectory() as d:
    t = time.perf_counter()
    sio.write_snapshot(os.path.join(d, "a.csv"), ids, pos, vel)
    native = time.perf_counter() - t
    t = time.perf_counter()
    sio.write_snapshot_npz(os.path.join(d, "a.npz"), ids, pos, vel)
    npz = time.perf_counter() - t
    t = time.perf_counter()
    sio.read_snapshot(os.path.join(d, "a.csv"))
    read = time.perf_counter() - t
m = min(n, 100_000)  # the python loop on a sample, scaled
t = time.perf_counter()
lines = [sio.SNAPSHOT_HEADER]
for i in range(m):
    x, y, z = pos[i]
    vx, vy, vz = vel[i]
    lines.append(f"{int(ids[i])},{x:.17g},{y:.17g},{z:.17g},"
                 f"{vx:.17g},{vy:.17g},{vz:.17g}")
"\n".join(lines)
py = (time.perf_counter() - t) * n / m
print(f"rows {n}: native csv {native:.3f} s ({n / native / 1e6:.2f} Mrow/s, "
      f"{sio._threads()} threads), reference loop {py:.2f} s "
      f"(x{py / native:.1f}), npz {npz:.3f} s, csv read {read:.2f} s")
