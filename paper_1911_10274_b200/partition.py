"""Mass-range partition of one store across ranks (config E: a single giant
lattice over 8 GPUs).

Rank r owns the mass slots ``[cuts[r], cuts[r+1])``.  Its shard holds

* its owned masses, then the *ghost* masses it needs -- every mass that
  shares a spring with an owned mass but is owned elsewhere -- in ascending
  global slot order;
* every spring slot with at least one owned endpoint, in ascending GLOBAL
  slot order.  Each owned mass therefore sees exactly its own springs in
  the reference's accumulation order (kernels.py:36, 71-76), so an owned
  mass's force -- and its whole trajectory -- is bit-identical to the
  unpartitioned run in fp64;
* ghosts are marked fixed + ghost: never integrated, their positions are
  overwritten before every step by the halo exchange, and spring side
  effects (break / zero-length counters) are only counted where the m1
  endpoint is owned, so the per-rank counters add up to the global ones.

Row-major lattice ids make mass ranges x-slabs (builder.py:124-125): the
halo of a slab is one plane of masses per neighbouring slab.

The exchange moves positions only (ghost velocities are never read: contact
and friction are evaluated for owned masses only).  ``HaloPlan`` is pure
index bookkeeping (numpy); ``exchange`` runs it over torch.distributed --
NCCL on GPUs, gloo in the CPU tests.  No collective appears anywhere else
on the step path.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

MASS_KEYS = ("m_pos", "m_vel", "m_acc", "m_fext", "m_load", "m_mass",
             "m_fixed", "m_alive", "m_gen")
SPRING_KEYS = ("s_m1", "s_m2", "s_m1gen", "s_m2gen", "s_rest", "s_k",
               "s_diam", "s_yield", "s_mode", "s_amp", "s_freq", "s_off",
               "s_per", "s_alive", "s_degen")


def even_cuts(m_n: int, ranks: int, align: int = 1) -> list[int]:
    """Equal mass ranges (optionally aligned, e.g. to lattice planes)."""
    per = -(-m_n // ranks)
    per = -(-per // align) * align
    cuts = [min(m_n, r * per) for r in range(ranks)] + [m_n]
    return cuts


@dataclass
class Shard:
    rank: int
    lo: int
    hi: int
    local_to_global: np.ndarray      # local mass index -> global slot
    spring_slots: np.ndarray         # local spring index -> global slot
    n_owned: int
    ghost_local: np.ndarray          # local indices of the ghosts
    ghost_owner: np.ndarray          # owning rank of each ghost
    case: dict = field(repr=False)   # rank-local case (oracle/ABI layout)

    @property
    def owned_local(self) -> np.ndarray:
        return np.arange(self.n_owned)


@dataclass
class HaloPlan:
    """Who sends which owned positions to whom.  ``send[q]`` = local
    indices (this rank) to send to rank q, in the order rank q lists the
    matching ghosts in ``recv[q]`` (its local indices)."""
    rank: int
    send: dict
    recv: dict

    @property
    def peers(self) -> list[int]:
        return sorted(set(self.send) | set(self.recv))


def partition_case(case: dict, cuts: list[int],
                   ranks: list[int] | None = None) -> list[Shard]:
    """Split a case dict (store arrays, golden/ABI layout) by mass ranges.
    With ``ranks``, only those shards carry their sub-case (``case``); the
    others are index bookkeeping only (enough for ``halo_plans``) -- one
    rank of a big partitioned run builds just its own arrays."""
    m_n = len(case["m_mass"])
    s1 = np.asarray(case["s_m1"], np.int64)
    s2 = np.asarray(case["s_m2"], np.int64)
    owner = np.searchsorted(np.asarray(cuts[1:]), np.arange(m_n),
                            side="right")
    shards = []
    for r in range(len(cuts) - 1):
        lo, hi = cuts[r], cuts[r + 1]
        own1 = (s1 >= lo) & (s1 < hi)
        own2 = (s2 >= lo) & (s2 < hi)
        sel = np.flatnonzero(own1 | own2)            # ascending global slot
        ends = np.concatenate([s1[sel], s2[sel]])
        ghosts = np.unique(ends[(ends < lo) | (ends >= hi)])
        l2g = np.concatenate([np.arange(lo, hi, dtype=np.int64), ghosts])
        if ranks is not None and r not in ranks:
            shards.append(Shard(rank=r, lo=lo, hi=hi, local_to_global=l2g,
                                spring_slots=sel, n_owned=hi - lo,
                                ghost_local=np.arange(hi - lo, len(l2g)),
                                ghost_owner=owner[ghosts], case=None))
            continue
        g2l = np.full(m_n, -1, np.int64)
        g2l[l2g] = np.arange(len(l2g))
        sub = {}
        for k in MASS_KEYS:
            sub[k] = np.array(np.asarray(case[k])[l2g], copy=True)
        n_own = hi - lo
        sub["m_fixed"] = sub["m_fixed"].astype(np.uint8)
        sub["m_fixed"][n_own:] = 1                   # ghosts: never integrated
        for k in SPRING_KEYS:
            sub[k] = np.array(np.asarray(case[k])[sel], copy=True)
        sub["s_m1"] = g2l[s1[sel]]
        sub["s_m2"] = g2l[s2[sel]]
        for k in ("gravity", "drag", "planes", "balls", "gc_kind", "gc_vec"):
            if k in case:
                sub[k] = case[k]
        # local-constraint CSR restricted to the shard's masses
        if "lc_off" in case:
            off = np.asarray(case["lc_off"], np.int64)
            kind = np.asarray(case["lc_kind"])
            vec = np.asarray(case["lc_vec"]).reshape(-1, 3)
            cnt = off[l2g + 1] - off[l2g]
            new_off = np.zeros(len(l2g) + 1, np.int64)
            np.cumsum(cnt, out=new_off[1:])
            rows = np.concatenate([np.arange(off[g], off[g + 1])
                                   for g in l2g]) if len(l2g) else \
                np.zeros(0, np.int64)
            rows = rows.astype(np.int64)
            sub["lc_off"] = new_off
            sub["lc_kind"] = kind[rows] if len(rows) else kind[:0]
            sub["lc_vec"] = vec[rows] if len(rows) else vec[:0]
        shards.append(Shard(rank=r, lo=lo, hi=hi, local_to_global=l2g,
                            spring_slots=sel, n_owned=n_own,
                            ghost_local=np.arange(n_own, len(l2g)),
                            ghost_owner=owner[ghosts], case=sub))
    return shards


def halo_plans(shards: list[Shard]) -> list[HaloPlan]:
    plans = [HaloPlan(rank=s.rank, send={}, recv={}) for s in shards]
    for s in shards:
        ghosts_g = s.local_to_global[s.ghost_local]
        for q in np.unique(s.ghost_owner).tolist():
            pick = s.ghost_owner == q
            plans[s.rank].recv[q] = s.ghost_local[pick]
            # the owner's local index of a global slot is slot - lo
            plans[q].send[s.rank] = ghosts_g[pick] - shards[q].lo
    return plans


def exchange(plan: HaloPlan, pos, dist=None, group=None):
    """One halo exchange of positions.  ``pos`` is a torch tensor of local
    position rows (any float dtype, >= 3 columns; device or host).  Sends
    pos[send[q], :3] to every peer q and writes what arrives into
    pos[recv[q], :3].  Point-to-point only (batched isend/irecv)."""
    import torch
    if dist is None:
        import torch.distributed as dist
    ops, inbox = [], {}
    dev = pos.device
    # fp32 contexts expose (record, low part) pairs (distributed._HiLo)
    split = hasattr(pos, "rows")
    cols = 6 if split else 3
    for q in plan.peers:
        if q in plan.send:
            idx = torch.as_tensor(plan.send[q], device=dev)
            rows = pos.rows(idx) if split else pos[idx, :3]
            ops.append(dist.P2POp(dist.isend, rows.contiguous(), q, group))
        if q in plan.recv:
            buf = torch.empty((len(plan.recv[q]), cols), dtype=pos.dtype,
                              device=dev)
            inbox[q] = buf
            ops.append(dist.P2POp(dist.irecv, buf, q, group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    for q, buf in inbox.items():
        idx = torch.as_tensor(plan.recv[q], device=dev)
        if split:
            pos.set_rows(idx, buf)
        else:
            pos[idx, :3] = buf
    return pos


def gather_owned(shards: list[Shard], key: str, parts: list[np.ndarray],
                 m_n: int) -> np.ndarray:
    """Reassemble a per-mass field from the owned rows of each shard."""
    out = np.zeros((m_n,) + parts[0].shape[1:], parts[0].dtype)
    for s, p in zip(shards, parts):
        out[s.lo:s.hi] = p[:s.n_owned]
    return out


def halo_dst_table(plans: list[HaloPlan], rank: int, n_local: int):
    """The in-library halo's send table of ``rank`` (sl_halo_init): int32
    [n_local, 2], entry (row << 3) | peer for each peer that holds this
    mass as a ghost -- peer = index in ``plans[rank].peers``, row = the
    ghost's local index there (``plans[q].recv[rank]`` lists them in the
    order of ``plans[rank].send[q]``) -- and -1 elsewhere.  Returns (table,
    peers, slots): slots[p] = this rank's counter slot at peer p (its
    index in that peer's peer list)."""
    plan = plans[rank]
    peers = plan.peers
    if len(peers) > 8:
        raise ValueError("at most 8 halo peers per rank")
    dst = np.full((n_local, 2), -1, np.int32)
    for p, q in enumerate(peers):
        if q not in plan.send:
            continue
        src = np.asarray(plan.send[q], np.int64)
        rows = np.asarray(plans[q].recv[rank], np.int64)
        if len(src) != len(rows):
            raise ValueError("halo plans disagree")
        if len(rows) and rows.max() >= (1 << 28):
            raise ValueError("ghost row index too large for the halo table")
        code = (rows << 3 | p).astype(np.int32)
        free = (dst[src, 0] < 0).astype(np.int64)  # first free column
        col = np.where(free == 1, 0, 1)
        if np.any(dst[src[col == 1], 1] >= 0):
            raise ValueError("a mass is a ghost of more than two peers")
        dst[src, col] = code
    slots = [plans[q].peers.index(rank) for q in peers]
    return dst, peers, slots
