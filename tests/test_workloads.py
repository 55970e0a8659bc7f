"""oracle/workloads.py (numpy-only bench inputs of the reference arm) ==
the product builder's stores, array for array -- so the reference arm and
the GPU arm step the same workload while the reference arm maps nothing
from the product package."""
import numpy as np
import pytest

import bench
import workloads as wl

KEYS = ("m_pos", "m_mass", "s_m1", "s_m2", "s_rest", "s_k", "s_diam",
        "s_mode", "s_amp", "s_freq", "s_off", "s_per", "planes", "gravity")


def _same(case, st, env):
    got = bench.store_case(st, env)
    for k in KEYS:
        a, b = np.asarray(case[k]), np.asarray(got[k])
        if k == "s_per" and not case["s_mode"].any():
            continue  # period of unactuated springs is never read
        assert a.shape == b.shape, k
        assert a.tobytes() == b.astype(a.dtype).tobytes(), k
    assert float(case["drag"]) == float(got["drag"])


@pytest.mark.parametrize("n", [3, 17, 24])
def test_config_b(n):
    _same(wl.config_b(n), *bench.build_workload(n))


def test_config_a():
    _same(wl.config_a(), *bench.build_cube())


@pytest.mark.parametrize("count,first", [(7, 0), (5, 3)])
def test_config_d(count, first):
    _same(wl.config_d(count, first), *bench.build_robots(count, first))
