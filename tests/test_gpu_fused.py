"""Multi-step fused small-body kernel (csrc/sl_fused.cuh, k_fused_small):
robot swarms run all the steps of an sl_step call in one launch with the
bodies' state in shared memory.  Checked against the per-step kernels
(SL_DISABLE_FUSED=1) and the reference oracle, through the C ABI; the
abort path (a zero-length spring appears) must commit nothing and re-run
the steps through the per-step kernels, which own the reference's event
semantics.
"""
import os

import numpy as np
import pytest

import oracle as orc
from conftest import rel_maxnorm
from test_gpu_window import _lattice_case

pytestmark = pytest.mark.gpu


def _ctx(case, fused=True):
    from conftest import case_context
    old = os.environ.get("SL_DISABLE_FUSED")
    os.environ["SL_DISABLE_FUSED"] = "0" if fused else "1"
    try:
        return case_context(case, "fp32")
    finally:
        if old is None:
            del os.environ["SL_DISABLE_FUSED"]
        else:
            os.environ["SL_DISABLE_FUSED"] = old


def _run(case, times, dt, fused, chunks=(None,), kill=None):
    ctx = _ctx(case, fused)
    c = np.zeros(3, np.int64)
    bounds = [0] + [b for b in chunks if b] + [len(times)]
    for q in range(len(bounds) - 1):
        if kill is not None and q == 1:
            ctx.kill_springs(kill.astype(np.int64))
        done, err = ctx.step(times[bounds[q]:bounds[q + 1]], dt, 0, c)
        assert err == 0
    st = ctx.stats()
    m, s = len(case["m_mass"]), len(case["s_m1"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    acc = np.zeros((m, 3))
    ctx.download_masses(pos, vel, acc)
    alive = np.zeros(s, np.uint8)
    degen = np.zeros(s, np.uint8)
    ctx.download_springs(alive, degen)
    ctx.close()
    return dict(pos=pos, vel=vel, acc=acc, alive=alive, degen=degen, c=c,
                st=st)


def _oracle(case, times, dt, kill=None, kill_at=None):
    ref = orc.OracleSim(case)
    for n in range(len(times)):
        if kill is not None and n == kill_at:
            ref.c["s_alive"][kill] = 0
        ref.step(float(times[n]), dt)
    return ref.c


@pytest.mark.parametrize("worm", [False, True])
def test_fused_robots_match_per_step_and_oracle(worm):
    case = _lattice_case(0, 0, 0, robots=11, worm=worm)
    dt, n = 1e-4, 100
    times = np.arange(n, dtype=np.float64) * dt
    f = _run(case, times, dt, True, chunks=(50,))
    p = _run(case, times, dt, False, chunks=(50,))
    assert f["st"]["fused_groups"] > 0 and f["st"]["fused_launches"] == 2
    assert f["st"]["fused_aborts"] == 0
    assert p["st"]["fused_groups"] == 0
    # same entry arithmetic and order as the window kernel
    assert rel_maxnorm(f["pos"], p["pos"]) < 1e-6
    assert rel_maxnorm(f["vel"], p["vel"]) < 1e-5
    assert rel_maxnorm(f["acc"], p["acc"]) < 1e-4
    assert np.array_equal(f["alive"], p["alive"])
    ref = _oracle(case, times, dt)
    assert rel_maxnorm(f["pos"], ref["m_pos"]) < 1e-4
    # north_star fp32 contract over the 100-step horizon (compensated
    # positions)
    assert rel_maxnorm(f["vel"], ref["m_vel"]) < 1e-4


@pytest.mark.parametrize("big", [False, True])
def test_fused_kills_between_launches(big):
    # robots: 512-thread groups; big: the 10^3 cube in one 1024-thread group
    case = _lattice_case(10, 10, 10) if big else \
        _lattice_case(0, 0, 0, robots=6)
    dt, n = 1e-4, 90
    times = np.arange(n, dtype=np.float64) * dt
    rng = np.random.default_rng(3)
    kill = np.sort(rng.choice(len(case["s_m1"]), 300, replace=False))
    f = _run(case, times, dt, True, chunks=(40,), kill=kill)
    p = _run(case, times, dt, False, chunks=(40,), kill=kill)
    assert f["st"]["fused_launches"] == 2
    assert rel_maxnorm(f["pos"], p["pos"]) < 1e-6
    assert np.array_equal(f["alive"], p["alive"])
    ref = _oracle(case, times, dt, kill=kill, kill_at=40)
    assert rel_maxnorm(f["pos"], ref["m_pos"]) < 1e-4


def test_fused_abort_reruns_per_step():
    """Two coincident masses joined by a spring: the fast path's sum is
    non-finite at the first step, the fused launch aborts without
    committing, and the per-step kernels produce the reference's
    zero-length semantics (flag + counter, no force)."""
    case = _lattice_case(0, 0, 0, robots=3)
    m1, m2 = int(case["s_m1"][0]), int(case["s_m2"][0])
    case["m_pos"] = case["m_pos"].copy()
    case["m_pos"][m2] = case["m_pos"][m1]
    dt, n = 1e-4, 30
    times = np.arange(n, dtype=np.float64) * dt
    f = _run(case, times, dt, True)
    p = _run(case, times, dt, False)
    assert f["st"]["fused_aborts"] == 1
    assert f["pos"].tobytes() == p["pos"].tobytes()
    assert f["vel"].tobytes() == p["vel"].tobytes()
    assert np.array_equal(f["degen"], p["degen"])
    assert f["c"].tolist() == p["c"].tolist()
    assert f["degen"][0] == 1


@pytest.mark.parametrize("dims", [(10, 10, 10), (9, 11, 8), (12, 9, 9)])
def test_fused_large_body_1024_threads(dims):
    """A single body of 513..1024 masses (the config-A 10^3 cube) runs in
    the 1024-thread variant: one CTA holds the whole body for all steps."""
    case = _lattice_case(*dims)
    dt, n = 1e-4, 80
    times = np.arange(n, dtype=np.float64) * dt
    f = _run(case, times, dt, True, chunks=(30,))
    p = _run(case, times, dt, False, chunks=(30,))
    assert f["st"]["fused_groups"] == 1 and f["st"]["fused_launches"] == 2
    assert f["st"]["fused_aborts"] == 0
    assert rel_maxnorm(f["pos"], p["pos"]) < 1e-6
    assert rel_maxnorm(f["vel"], p["vel"]) < 1e-5
    assert np.array_equal(f["alive"], p["alive"])
    ref = _oracle(case, times, dt)
    assert rel_maxnorm(f["pos"], ref["m_pos"]) < 1e-4
    assert rel_maxnorm(f["vel"], ref["m_vel"]) < 1e-4
