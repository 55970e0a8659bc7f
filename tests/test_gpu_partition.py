"""Partitioned runs on the device (config E path), all shards on cuda:0.

Each shard is its own context (owned masses + ghosts, ghosts marked);
before every step the halo exchange rewrites ghost rows of the position
buffer the step reads, on the context streams; steps are enqueued
asynchronously.  fp64 partitioned trajectories must equal the single
context BIT FOR BIT, spring events must add up to the single run's
counters (ghost-side events are not double counted), and the fp32 split
layout must stay within tolerance.  The cross-GPU transport (NCCL
batched isend/irecv) is the same `partition.exchange` the gloo test
(tests/test_partition.py) runs between processes.
"""
import numpy as np
import pytest
import torch

from conftest import load_golden, rel_maxnorm
from paper_1911_10274_b200 import _native
from paper_1911_10274_b200.distributed import (PartitionedRun,
                                               context_for_case,
                                               position_view)
from paper_1911_10274_b200.partition import (even_cuts, halo_plans,
                                             partition_case)
from test_partition import lattice_case

pytestmark = pytest.mark.gpu


def single(case, steps, dt, precision="fp64"):
    ctx = context_for_case(case, 0, precision)
    c = np.zeros(3, np.int64)
    done, err = ctx.step(np.arange(steps) * dt, dt, 0, c)
    m, s = len(case["m_mass"]), len(case["s_m1"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    alive = np.zeros(s, np.uint8)
    ctx.download_springs(alive)
    ctx.close()
    return pos, vel, alive, c


def partitioned(case, ranks, steps, dt, precision="fp64"):
    m_n = len(case["m_mass"])
    shards = partition_case(case, even_cuts(m_n, ranks))
    plans = halo_plans(shards)
    runs = [PartitionedRun(s, p, 0, precision) for s, p in
            zip(shards, plans)]
    views = {}
    for n in range(steps):
        # current read buffers of every shard, then the exchange between
        # them (device copies), then every shard's step
        for r, run in enumerate(runs):
            views[r] = position_view(run.ctx)
        torch.cuda.synchronize()
        for p in plans:
            for q, idx in p.recv.items():
                src = torch.as_tensor(plans[q].send[p.rank], device="cuda")
                dst = torch.as_tensor(idx, device="cuda")
                if hasattr(views[q], "rows"):  # fp32: record + low part
                    views[p.rank].set_rows(dst, views[q].rows(src))
                else:
                    views[p.rank][dst, :3] = views[q][src, :3]
        torch.cuda.synchronize()
        for r, run in enumerate(runs):
            run.ctx.step_async(np.array([n * dt]), dt, _native.ACC_GATHER)
    pos = np.zeros((m_n, 3))
    vel = np.zeros((m_n, 3))
    alive = np.zeros(len(case["s_m1"]), np.uint8)
    counters = np.zeros(3, np.int64)
    for s, run in zip(shards, runs):
        done, err = run.finish()
        assert err == 0 and done == steps
        p, v, a = run.owned_state()
        pos[s.lo:s.hi], vel[s.lo:s.hi] = p, v
        alive[s.spring_slots] = a     # crossing springs agree (asserted)
        counters += run.counters
        run.close()
    return pos, vel, alive, counters


@pytest.mark.parametrize("ranks", [2, 3])
def test_partitioned_fp64_bit_exact(ranks):
    case = lattice_case(8, 5, 4)
    want = single(case, 60, 1e-4)
    got = partitioned(case, ranks, 60, 1e-4)
    assert got[0].tobytes() == want[0].tobytes()
    assert got[1].tobytes() == want[1].tobytes()


def test_partitioned_yield_breaks_count_once():
    g = load_golden("yield_break")
    case = dict(g)
    steps, dt = int(g["n_steps"]), float(g["dt"])
    want = single(case, steps, dt)
    got = partitioned(case, 2, steps, dt)
    assert np.array_equal(got[2], want[2])          # same springs broke
    assert got[3].tolist() == want[3].tolist()      # counted once
    assert got[0].tobytes() == want[0].tobytes()


def test_partitioned_fp32_split_within_tolerance():
    case = lattice_case(8, 5, 4)
    want = single(case, 60, 1e-4)
    got = partitioned(case, 2, 60, 1e-4, "fp32")
    assert rel_maxnorm(got[0], want[0]) < 1e-6
    assert rel_maxnorm(got[1], want[1]) < 1e-4
