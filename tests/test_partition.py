"""Mass-range partition + halo exchange (config E host logic), on CPU.

The stepping here is the oracle (the reference algorithm) run per shard --
the same Shard / HaloPlan / exchange code the GPU path drives
(paper_1911_10274_b200/partition.py, distributed.py).  Partitioned runs
must equal the single run BIT FOR BIT (fp64): each owned mass sees its
springs in global slot order and exact copies of its ghosts' positions.
The 2-rank test exchanges over torch.distributed with the gloo backend.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, Vec3)
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
from paper_1911_10274_b200.partition import (even_cuts, exchange,
                                             gather_owned, halo_plans,
                                             partition_case)
from test_host_parity import our_case

STEPS, DT = 40, 1e-4


def lattice_case(nx=6, ny=5, nz=4):
    st = ObjectStore()
    build_lattice(LatticeSpec(Vec3(0, 0, -0.004), nx, ny, nz, 0.05,
                              Material(1e5, 1000.0)), st)
    st._m_pos[:st.mass_slot_count] *= 1.03
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01, contacts=[
        ContactPlane(normal=Vec3(0, 0, 1), offset=0.0, stiffness=800.0,
                     static_friction=0.7, kinetic_friction=0.5)])
    return {k: np.array(v, copy=True) for k, v in our_case(st, env).items()}


def single_run(case):
    ref = orc.OracleSim(case)
    ref.run(STEPS, DT, time_rule="index")
    return ref.c["m_pos"], ref.c["m_vel"]


class LocalDist:
    """In-process stand-in for torch.distributed P2P between shard
    objects (each 'rank' is a tensor in one process)."""

    def __init__(self, tensors):
        self.t = tensors


def local_exchange(plans, pos_tensors):
    # what each rank would send, then delivered to the receivers
    for p in plans:
        for q, idx in p.recv.items():
            src = plans[q].send[p.rank]
            pos_tensors[p.rank][idx, :3] = pos_tensors[q][src, :3]


@pytest.mark.parametrize("ranks", [2, 3, 4])
def test_partitioned_oracle_equals_single_run(ranks):
    case = lattice_case()
    want_p, want_v = single_run(case)
    m_n = len(case["m_mass"])
    shards = partition_case(case, even_cuts(m_n, ranks))
    plans = halo_plans(shards)
    sims = [orc.OracleSim(s.case) for s in shards]
    pos_t = [torch.from_numpy(s.c["m_pos"]) for s in sims]
    for n in range(STEPS):
        local_exchange(plans, pos_t)
        for s in sims:
            s.step(n * DT, DT)
    got_p = gather_owned(shards, "m_pos", [s.c["m_pos"] for s in sims], m_n)
    got_v = gather_owned(shards, "m_vel", [s.c["m_vel"] for s in sims], m_n)
    assert got_p.tobytes() == want_p.tobytes()
    assert got_v.tobytes() == want_v.tobytes()


def test_partition_structure():
    case = lattice_case(8, 3, 3)
    m_n = len(case["m_mass"])
    cuts = even_cuts(m_n, 4, align=9)      # whole x-planes of 3x3
    shards = partition_case(case, cuts)
    plans = halo_plans(shards)
    seen = np.zeros(len(case["s_m1"]), np.int64)
    for s in shards:
        assert np.all(np.diff(s.spring_slots) > 0)      # global slot order
        seen[s.spring_slots] += 1
        assert np.all(s.case["m_fixed"][s.n_owned:] == 1)
        g = s.local_to_global[s.ghost_local]
        assert np.all((g < s.lo) | (g >= s.hi))
        # x-slab halo: one plane per neighbouring slab
        assert len(s.ghost_local) <= 2 * 9
    # crossing springs live in exactly two shards, the rest in one
    s1, s2 = case["s_m1"], case["s_m2"]
    owner = np.searchsorted(np.asarray(cuts[1:]), np.arange(m_n), "right")
    assert np.array_equal(seen, 1 + (owner[s1] != owner[s2]))
    for p in plans:
        for q, idx in p.send.items():
            assert len(idx) == len(plans[q].recv[p.rank])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, cuts, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shards = partition_case(case, cuts)
        plan = halo_plans(shards)[rank]
        sim = orc.OracleSim(shards[rank].case)
        pos = torch.from_numpy(sim.c["m_pos"])
        for n in range(STEPS):
            exchange(plan, pos)
            sim.step(n * DT, DT)
        own = torch.from_numpy(np.ascontiguousarray(
            np.concatenate([sim.c["m_pos"][:shards[rank].n_owned],
                            sim.c["m_vel"][:shards[rank].n_owned]], 1)))
        parts = [torch.zeros((s.n_owned, 6), dtype=torch.float64)
                 for s in shards]
        dist.all_gather(parts, own)
        if rank == 0:
            out.put(torch.cat(parts).numpy().tobytes())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_halo_equals_single_run():
    case = lattice_case()
    want_p, want_v = single_run(case)
    m_n = len(case["m_mass"])
    cuts = even_cuts(m_n, 2)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, cuts, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = np.frombuffer(q.get(timeout=120), np.float64).reshape(m_n, 6)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert got[:, :3].tobytes() == np.ascontiguousarray(want_p).tobytes()
    assert got[:, 3:].tobytes() == np.ascontiguousarray(want_v).tobytes()


@pytest.mark.parametrize("ranks", [2, 3, 5])
def test_halo_dst_table_reproduces_exchange(ranks):
    """The in-library halo's per-mass send table (partition.halo_dst_table,
    consumed by the step kernels through sl_halo_init) moves exactly the
    rows the HaloPlan exchange moves: every ghost row of every rank gets
    its owner's position, nothing else is written."""
    from paper_1911_10274_b200.partition import halo_dst_table
    case = lattice_case(8, 5, 4)
    m = len(case["m_mass"])
    cuts = even_cuts(m, ranks)
    shards = partition_case(case, cuts)
    plans = halo_plans(shards)
    rng = np.random.default_rng(ranks)
    truth = rng.normal(size=(m, 3))
    local = [np.full((len(s.local_to_global), 3), np.nan) for s in shards]
    for s, loc in zip(shards, local):
        loc[:s.n_owned] = truth[s.local_to_global[:s.n_owned]]
    for s in shards:
        dst, peers, slots = halo_dst_table(plans, s.rank,
                                           len(s.local_to_global))
        assert (dst[s.n_owned:] == -1).all()  # ghosts never send
        for i, j in zip(*np.nonzero(dst >= 0)):
            code = int(dst[i, j])
            q = peers[code & 7]
            local[q][code >> 3] = local[s.rank][i]
        for p, q in enumerate(peers):  # counter slots are mutual
            assert plans[q].peers[slots[p]] == s.rank
    for s, loc in zip(shards, local):
        assert np.array_equal(loc, truth[s.local_to_global])
