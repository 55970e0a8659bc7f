"""In-library halo of a mass-range partition (config E): the step kernels
store owned boundary positions straight into the peers' ghost rows, a
one-block kernel per step publishes and awaits per-peer step counters
(csrc/sl_device.cuh HaloDesc, sl_api.cu k_halo_sync).

* several shards in ONE process on one device (plain pointers between the
  contexts) == the unpartitioned run, bit for bit, in fp64 and fp32;
* two PROCESSES on one device through CUDA IPC mappings (the handles
  travel once over a gloo group) == the unpartitioned run, bit for bit.
The partition follows the row-major ids of the reference builder
(/root/reference/pkg/src/softlat/builder.py:124-125): mass ranges are
x-slabs."""
import os
import sys

import numpy as np
import pytest

from conftest import ROOT, case_context

pytestmark = pytest.mark.gpu


def _lattice(nx=12, ny=7, nz=6):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import workloads
    case = workloads.config_b(1)  # shape template
    pos = workloads.grid_positions((0.0, 0.0, 0.0), nx, ny, nz, 0.05)
    a, b = workloads.grid_springs(nx, ny, nz)
    rest, stiff, diam, mass = workloads.materialize(pos, a, b, 1e5, 1000.0,
                                                    1e-3)
    case = workloads.make_case(pos * 1.01, mass, a, b, rest, stiff, diam,
                               (0, 0, -9.81), workloads.ground(2000.0))
    return case, ny * nz


def _single(case, precision, steps, dt=1e-4):
    # the per-step kernels, as the shards run (ghosts rule out the fused
    # multi-step kernel, whose sum order differs)
    old = os.environ.get("SL_DISABLE_FUSED")
    os.environ["SL_DISABLE_FUSED"] = "1"
    try:
        ctx = case_context(case, precision)
    finally:
        if old is None:
            del os.environ["SL_DISABLE_FUSED"]
        else:
            os.environ["SL_DISABLE_FUSED"] = old
    c = np.zeros(3, np.int64)
    done, err = ctx.step(np.arange(steps) * dt, dt, 0, c)
    assert err == 0
    m = len(case["m_mass"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    ctx.close()
    return pos, vel


@pytest.mark.parametrize("precision", ["fp64", "fp32", "mixed"])
@pytest.mark.parametrize("ranks", [2, 3, 4])
def test_in_process_halo_bit_exact(ranks, precision):
    from paper_1911_10274_b200.distributed import HaloRun
    from paper_1911_10274_b200.partition import (even_cuts, halo_plans,
                                                 partition_case)
    case, plane = _lattice()
    m = len(case["m_mass"])
    cuts = even_cuts(m, ranks, align=plane)
    shards = partition_case(case, cuts)
    plans = halo_plans(shards)
    runs = [HaloRun(s, plans, 0, precision) for s in shards]
    HaloRun.connect_local(runs)
    steps, dt = 40, 1e-4
    times = np.arange(steps) * dt
    # enqueue every shard before any waits: the per-step counters order
    # the shards on the device, the host never blocks in between
    for k in range(0, steps, 10):
        for r in runs:
            r.step_async(times[k:k + 10], dt)
    pos = np.zeros((m, 3))
    vel = np.zeros((m, 3))
    for s, r in zip(shards, runs):
        done, err = r.finish()
        assert err == 0 and done == steps
        p, v, _ = r.owned_state()
        pos[s.lo:s.hi], vel[s.lo:s.hi] = p, v
        r.close()
    ref_p, ref_v = _single(case, precision, steps)
    assert pos.tobytes() == ref_p.tobytes()
    assert vel.tobytes() == ref_v.tobytes()


def _worker(rank, world, port, precision, steps, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1911_10274_b200.distributed import run_partitioned
    from paper_1911_10274_b200.partition import even_cuts
    case, plane = _lattice()
    cuts = even_cuts(len(case["m_mass"]), world, align=plane)
    shard, pos, vel, alive, counters, sec = run_partitioned(
        case, cuts, steps, 1e-4, precision, device=0)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), pos=pos, vel=vel,
             lo=shard.lo, hi=shard.hi)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["fp64", "fp32"])
def test_two_processes_ipc_halo_bit_exact(tmp_path, precision):
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    steps = 20
    mp.spawn(_worker, args=(2, port, precision, steps, str(tmp_path)),
             nprocs=2, join=True)
    case, _ = _lattice()
    m = len(case["m_mass"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    for r in range(2):
        z = np.load(tmp_path / f"r{r}.npz")
        pos[int(z["lo"]):int(z["hi"])] = z["pos"]
        vel[int(z["lo"]):int(z["hi"])] = z["vel"]
    ref_p, ref_v = _single(case, precision, steps)
    assert pos.tobytes() == ref_p.tobytes()
    assert vel.tobytes() == ref_v.tobytes()
