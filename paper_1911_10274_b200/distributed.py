"""Running one partitioned store across devices (config E) and independent
instances across ranks (configs B / D).

``PartitionedRun`` drives one shard (partition.py) on one device: its
context holds the owned masses plus ghosts; before every step the halo
exchange rewrites the ghost rows of the position buffer the step will read,
on the context's own CUDA stream, then the step is enqueued asynchronously
(sl_step_async).  The host never synchronises inside the run; the only
cross-rank traffic is the point-to-point halo (NCCL over NVLink on GPUs,
gloo in the CPU tests) -- no collective on the step path.

The position buffer is exposed to torch through
``__cuda_array_interface__`` (sl_state_pointers); torch is plumbing here:
the index gather / scatter of the halo rows and the NCCL calls.
"""
from __future__ import annotations

import numpy as np

from . import _native
from .partition import HaloPlan, Shard, exchange


def context_for_case(case: dict, device: int = 0, precision: str = "fp64",
                     v_stick: float = 1e-6) -> _native.Context:
    """A context loaded with a case dict (store arrays in the reference
    layout, e.g. a Shard.case or a golden case)."""
    ctx = _native.Context(device, precision)
    ctx.upload_masses(case["m_pos"], case["m_vel"], case["m_acc"],
                      case["m_fext"], case["m_load"], case["m_mass"],
                      case["m_fixed"], case["m_alive"], case["m_gen"])
    ctx.upload_springs(case["s_m1"], case["s_m2"], case["s_m1gen"],
                       case["s_m2gen"], case["s_rest"], case["s_k"],
                       case["s_diam"], case["s_yield"], case["s_mode"],
                       case["s_amp"], case["s_freq"], case["s_off"],
                       case["s_per"], case["s_alive"], case["s_degen"])
    n = len(case["m_mass"])
    ctx.set_local_constraints(case.get("lc_off", np.zeros(n + 1, np.int64)),
                              case.get("lc_kind", np.zeros(0, np.int8)),
                              case.get("lc_vec", np.zeros((0, 3))))
    ctx.set_environment(case["gravity"], float(np.asarray(case["drag"])),
                        case.get("planes", np.zeros((0, 7))),
                        case.get("balls", np.zeros((0, 5))),
                        case.get("gc_kind", np.zeros(0, np.int8)),
                        case.get("gc_vec", np.zeros((0, 3))), v_stick)
    return ctx


class _DeviceArray:
    def __init__(self, ptr: int, rows: int, record_bytes: int):
        self.__cuda_array_interface__ = {
            "shape": (rows, 2 if record_bytes == 8 else 4),
            "typestr": "<f8" if record_bytes == 32 else "<f4",
            "data": (ptr, False), "version": 2, "strides": None}


def position_view(ctx: _native.Context):
    """torch view of the buffer the next step reads: (rows, 4) = (x, y, z,
    m); in fp32 mode a pair: the records (x, y, z, lx) and the position low
    parts (ly, lz) (sl_state_lo) -- the halo moves all six.  Re-fetch after
    every step (the buffers ping-pong)."""
    import torch
    ptr, rows, rb = ctx.state_pointers()
    dev = f"cuda:{ctx.device}"
    hi = torch.as_tensor(_DeviceArray(ptr, rows, rb), device=dev)
    lo = ctx.state_lo()
    if not lo:
        return hi
    return _HiLo(hi, torch.as_tensor(_DeviceArray(lo, rows, 8), device=dev))


class _HiLo:
    """(record, low part) pair behind the exchange's row indexing."""

    def __init__(self, hi, lo):
        self.hi, self.lo = hi, lo
        self.device, self.dtype = hi.device, hi.dtype

    def rows(self, idx):
        import torch
        return torch.cat([self.hi[idx, :4], self.lo[idx, :2]], dim=1)

    def set_rows(self, idx, buf):
        self.hi[idx, :4] = buf[:, :4]
        self.lo[idx, :2] = buf[:, 4:6]


class PartitionedRun:
    """One shard of a mass-range partition on one device."""

    def __init__(self, shard: Shard, plan: HaloPlan, device: int = 0,
                 precision: str = "fp64", accumulation: int =
                 _native.ACC_GATHER):
        self.shard = shard
        self.plan = plan
        self.acc = accumulation
        self.ctx = context_for_case(shard.case, device, precision)
        if len(shard.ghost_local):
            self.ctx.mark_ghosts(shard.ghost_local)
        self.counters = np.zeros(3, np.int64)

    def stream(self):
        import torch
        return torch.cuda.ExternalStream(self.ctx.stream(),
                                         device=f"cuda:{self.ctx.device}")

    def step_async(self, sim_t: float, dt: float, halo) -> None:
        """Halo exchange then one step, both enqueued on the context
        stream.  ``halo(plan, pos_view)`` performs the exchange."""
        import torch
        with torch.cuda.stream(self.stream()):
            halo(self.plan, position_view(self.ctx))
        self.ctx.step_async(np.array([sim_t]), dt, self.acc)

    def finish(self) -> tuple[int, int]:
        return self.ctx.step_finish(self.counters)

    def owned_state(self):
        m = self.shard.n_owned
        n = len(self.shard.local_to_global)
        pos, vel = np.zeros((n, 3)), np.zeros((n, 3))
        self.ctx.download_masses(pos, vel)
        alive = np.zeros(len(self.shard.spring_slots), np.uint8)
        self.ctx.download_springs(alive)
        return pos[:m], vel[:m], alive

    def close(self):
        self.ctx.close()


class HaloRun:
    """One shard of a mass-range partition with the IN-LIBRARY halo
    (sl_halo_*): the owner's step kernel stores boundary positions straight
    into the peers' ghost rows over mapped peer memory, a one-block kernel
    per step publishes / awaits per-peer step counters.  A whole
    ``step(times)`` call is one library call: no Python, no torch, no
    collective on the step path.  ``connect_local`` wires shards that live
    in one process; ``connect_ipc`` wires one shard per process (CUDA IPC,
    the handles travel once over torch.distributed)."""

    def __init__(self, shard: Shard, plans: list, device: int = 0,
                 precision: str = "fp64"):
        from .partition import halo_dst_table
        self.shard = shard
        self.rank = shard.rank
        self.ctx = context_for_case(shard.case, device, precision)
        if len(shard.ghost_local):
            self.ctx.mark_ghosts(shard.ghost_local)
        dst, self.peers, self.slots = halo_dst_table(
            plans, shard.rank, len(shard.local_to_global))
        self.counters = np.zeros(3, np.int64)
        # build the device layout now (a zero-step call): nothing may
        # allocate (cudaMalloc can synchronise the device) once the
        # shards' step counters wait on one another
        self.ctx.step(np.zeros(0), 1e-4, _native.ACC_GATHER, self.counters)
        self.ctx.halo_init(len(self.peers), dst)

    @staticmethod
    def connect_local(runs: list["HaloRun"]):
        by_rank = {r.rank: r for r in runs}
        local = {r.rank: r.ctx.halo_local() for r in runs}
        for r in runs:
            for p, q in enumerate(r.peers):
                r.ctx.halo_set_peer(p, local[q], r.slots[p])
            r.ctx.halo_commit()
        return by_rank

    def connect_ipc(self, group=None):
        import torch.distributed as dist
        world = dist.get_world_size(group)
        mine = self.ctx.halo_ipc_handles()
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        for p, q in enumerate(self.peers):
            self.ctx.halo_set_peer(p, self.ctx.halo_ipc_open(allh[q]),
                                   self.slots[p])
        self.ctx.halo_commit()
        dist.barrier(group=group)

    def step(self, times: np.ndarray, dt: float,
             accumulation: int = _native.ACC_GATHER):
        return self.ctx.step(np.asarray(times, np.float64), dt, accumulation,
                             self.counters)

    def step_async(self, times: np.ndarray, dt: float,
                   accumulation: int = _native.ACC_GATHER):
        self.ctx.step_async(np.asarray(times, np.float64), dt, accumulation)

    def finish(self):
        return self.ctx.step_finish(self.counters)

    def owned_state(self):
        m = self.shard.n_owned
        n = len(self.shard.local_to_global)
        pos, vel = np.zeros((n, 3)), np.zeros((n, 3))
        self.ctx.download_masses(pos, vel)
        alive = np.zeros(len(self.shard.spring_slots), np.uint8)
        self.ctx.download_springs(alive)
        return pos[:m], vel[:m], alive

    def close(self):
        self.ctx.close()


def nccl_halo(plan: HaloPlan, pos, group=None):
    """Halo exchange over torch.distributed (NCCL between GPUs)."""
    return exchange(plan, pos, group=group)


def run_partitioned(case: dict, cuts: list[int], steps: int, dt: float,
                    precision: str = "fp64", device: int | None = None):
    """Multi-process driver (one rank per GPU, torchrun): this rank's shard
    of ``case`` stepped ``steps`` times with the in-library halo (CUDA IPC
    peer mappings; torch.distributed only carries the handles once).
    Returns (shard, owned positions, owned velocities, spring alive flags,
    counters, device seconds of the step kernels)."""
    import torch
    import torch.distributed as dist
    from .partition import halo_plans, partition_case
    rank = dist.get_rank()
    shards = partition_case(case, cuts)
    plans = halo_plans(shards)
    dev = torch.cuda.current_device() if device is None else device
    run = HaloRun(shards[rank], plans, dev, precision)
    run.connect_ipc()
    times = np.arange(steps, dtype=np.float64) * dt
    dist.barrier()
    run.ctx.sync()
    done, err = run.step(times, dt)
    sec = run.ctx.last_step_ms() / 1e3
    pos, vel, alive = run.owned_state()
    return shards[rank], pos, vel, alive, run.counters.copy(), sec
