"""Golden snapshot text made by the REFERENCE's own formatter.

Run in the build container only (needs /root/reference):

    python tests/golden/make_io_golden.py

Imports ``softlat.io`` from /root/reference/pkg/src, formats a seeded set of
rows chosen to stress "{:.17g}" (random magnitudes over the whole exponent
range, subnormals, +-0, integers, 17-digit boundaries, inf, -inf, nan, large
and negative ids) with ``io.format_snapshot`` (io.py:19-27) and stores the
inputs and the exact bytes in snapshot_io.npz.  Nothing on the GPU box reads
/root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/softlat_numba_cache")


def rows():
    rng = np.random.default_rng(20191122)
    n = 1000
    mant = rng.uniform(-10, 10, (n, 6))
    expo = rng.integers(-320, 309, (n, 6)).astype(np.float64)
    with np.errstate(over="ignore", under="ignore"):
        wild = mant * np.power(10.0, expo)
    plain = rng.normal(0, 1, (n, 6)) * rng.choice([1e-6, 1e-2, 1, 1e3, 1e9],
                                                   (n, 1))
    special = np.array([
        [0.0, -0.0, 1.0, -1.0, 0.1, 0.2],
        [5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
         -1.7976931348623157e308, 1e-5],
        [1e16, 1e17, 123456789012345678.0, 0.30000000000000004, 1e-4,
         9.999999999999999e-5],
        [np.inf, -np.inf, np.nan, -np.nan, 1e22, 1e-7],
        [2.0 ** 53, 2.0 ** 53 + 2, 0.5, 1.5e300, 3.0, 100.0],
    ])
    vals = np.concatenate([special, wild, plain])
    ids = np.concatenate([[0, 1, -5, 2 ** 62, -(2 ** 63)],
                          rng.integers(0, 2 ** 40, len(vals) - 5)])
    return ids.astype(np.int64), vals[:, :3].copy(), vals[:, 3:].copy()


def main():
    sys.path.insert(0, REF)
    from softlat import io as ref_io
    ids, pos, vel = rows()
    text = ref_io.format_snapshot(ids, pos, vel)
    empty = ref_io.format_snapshot(np.zeros(0, np.int64), np.zeros((0, 3)),
                                   np.zeros((0, 3)))
    np.savez_compressed(os.path.join(HERE, "snapshot_io.npz"), ids=ids,
                        pos=pos, vel=vel,
                        text=np.frombuffer(text.encode("ascii"), np.uint8),
                        empty=np.frombuffer(empty.encode("ascii"), np.uint8))
    print("rows", len(ids), "bytes", len(text))


if __name__ == "__main__":
    main()
