#!/usr/bin/env python
"""Throughput benchmark of the spring-mass step (BASELINE.json metric).

Default workload = config B of BASELINE.json / SURVEY.md 8(d): a 100^3
lattice (1,000,000 masses, 12,731,796 springs), spacing 0.05, E=1e5,
rho=1000, positions stretched x1.01 (the reference bench recipe,
cli.py:263-271), gravity -9.81 and a friction ground plane (k=2000,
mu_s=1, mu_k=0.8) with the bottom layer on it; fp32, deterministic gather.

One "step" = one fused spring+mass step of the whole lattice.  ``value`` =
alive springs x steps / device time (CUDA events on the library's stream,
max over ranks); ``e2e`` = the same metric through the public API
(SimController.start(duration) -> wait_for_event -> snapshot) with the host
store authoritative before and after, host<->device copies inside the timed
region.  Multi-GPU (torchrun): one independent lattice per rank (batched
instances, no collective on the step path; scaling "weak").

``--impl reference`` times the reference algorithm on the host CPU (the C
restatement in oracle/, OpenMP, all cores, fp64 slotted accumulation -- the
reference's fastest CPU variant) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PAPER_RATE = 3.0e8  # PAPER.md:10,20 headline (Titan X); north_star x50 base


def parse():
    args = _parser().parse_args()
    if args.n is None:
        args.n = 200 if args.config == "E" else 100
    return args


def _parser():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="B",
                    choices=["A", "B", "D", "E"],
                    help="B: one 100^3 lattice per rank (batched instances);"
                         " D: --robots actuated 5^3 robots sharded over "
                         "the ranks (RL batch); A: the reference's bouncing "
                         "10^3 cube (scenarios/bouncing_cube.ini) per rank;"
                         " E: ONE --edge^3 lattice (default 200) split by "
                         "mass range (x-slabs) over the ranks, in-library "
                         "halo over mapped peer memory")
    ap.add_argument("--n", "--edge", dest="n", type=int, default=None,
                    help="lattice edge (--edge under torchrun, whose parser "
                         "reads --n as ambiguous); 100, or 200 for E")
    ap.add_argument("--robots", type=int, default=4096)
    ap.add_argument("--precision", default="fp32",
                    choices=["fp32", "mixed", "fp64"])
    ap.add_argument("--accumulation", default="gather",
                    choices=["gather", "atomic"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp64", action="store_true",
                    help="skip the fp64 parity-mode sub-measurement")
    return ap


# --------------------------------------------------------------- workload
def build_workload(n: int):
    from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                       ObjectStore, Vec3)
    from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
    st = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0), n, n, n, 0.05,
                                     Material(1e5, 1000.0)), st)
    st._m_pos[body.mass_handles.slots] *= 1.01
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env


def build_cube():
    """Config A (scenarios/bouncing_cube.ini): a 10^3
    lattice, corner (0, 0, 0.3), spacing 0.1, E = 1e6, rho = 1000, d = 1 mm,
    falling onto a ground plane k = 2000, mu_s = 1, mu_k = 0.8."""
    from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                       ObjectStore, Vec3)
    from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
    st = ObjectStore()
    build_lattice(LatticeSpec(Vec3(0, 0, 0.3), 10, 10, 10, 0.1,
                              Material(1e6, 1000.0), 1e-3), st)
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=2000.0,
        static_friction=1.0, kinetic_friction=0.8)])
    return st, env


def build_robots(count: int, first: int = 0):
    """Config D: 5^3 robots, spacing 0.05, E = 1e6,
    worm-actuated (configure_worm), stacked along y as cmd_swarm does
    (cli.py:323-331), on a ground plane k = 500 with drag 0.01.  ``first``
    offsets this rank's shard so shards tile the global swarm."""
    from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                       ObjectStore, Vec3)
    from paper_1911_10274_b200.builder import LatticeSpec, build_robot_swarm
    st = ObjectStore()
    build_robot_swarm(LatticeSpec(Vec3(0, 0, 0), 5, 5, 5, 0.05,
                                  Material(1e6, 1000.0)), st, count,
                      first=first)
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01,
                      contacts=[ContactPlane(
                          normal=Vec3(0, 0, 1), offset=0.0, stiffness=500.0,
                          static_friction=1.0, kinetic_friction=0.8)])
    return st, env


def describe(args, world: int):
    """(workload description, scaling, per-spring extra words)."""
    if args.config == "D":
        return (f"D: {args.robots} worm-actuated 5^3 robots (RL batch) on a "
                f"friction ground plane, sharded over {world} rank(s), "
                f"{args.precision}, {args.accumulation}",
                "strong" if world > 1 else "weak", 1)
    if args.config == "A":
        return (f"A: 10^3 bouncing cube (scenarios/bouncing_cube.ini) per "
                f"rank, {args.precision}, {args.accumulation}", "weak", 0)
    if args.config == "E":
        return (f"E: one {args.n}^3 lattice (x1.01 stretch, gravity, "
                f"friction ground plane) split into {world} x-slab(s), "
                f"in-library halo, {args.precision}, {args.accumulation}",
                "strong", 0)
    return (f"B: {args.n}^3 lattice on friction ground plane, gravity, "
            f"x1.01 stretch, {args.precision}, {args.accumulation}",
            "weak", 0)


def make_workload(args, rank: int, world: int):
    """(store, env, description, scaling, per-spring extra words)."""
    desc, scaling, extra = describe(args, world)
    if args.config == "D":
        per = args.robots // world
        first = rank * per + min(rank, args.robots % world)
        count = per + (1 if rank < args.robots % world else 0)
        st, env = build_robots(count, first)
    elif args.config == "A":
        st, env = build_cube()
    else:
        st, env = build_workload(args.n)
    return st, env, desc, scaling, extra


def algorithmic_bytes(springs: int, masses: int, precision: str,
                      extra_words: int = 0) -> int:
    """B = S*Bs + M*Bm.  Bs = int32 i,j + k, L0 words (+ an
    actuation phase word for actuated springs); Bm = pos r+w, vel r+w, m r
    (words of the state precision).  The fp32 mode's positions are
    compensated (hi + lo): 6 position words r+w, so
    Bm = (12 + 6 + 1) x 4 = 76 B."""
    w_s = 8 if precision == "fp64" else 4
    if precision == "fp32":
        bm = 19 * 4
    else:
        bm = 13 * 8
    return springs * (8 + (2 + extra_words) * w_s) + masses * bm


# untimed control segments before the timed e2e one: the snapshot pool
# pages in (page-locked) buffer sets in the background during the first
# ones, and page-locking stalls the process's CUDA calls while it runs
E2E_WARM = int(os.environ.get("SL_E2E_WARM", "3"))
E2E_REPS = 5


def _native_pinned_copy(a):
    """A page-locked copy of a host array (the inputs of an e2e segment live
    in pinned memory, as the contract's host buffers)."""
    from paper_1911_10274_b200 import _native
    out = _native.pinned_empty(a.shape, a.dtype)
    out[...] = a
    return out


def store_case(st, env):
    from paper_1911_10274_b200 import engine
    m, s = st.mass_slot_count, st.spring_slot_count
    case = {k: getattr(st, "_" + k)[:m] for k in
            ("m_pos", "m_vel", "m_acc", "m_fext", "m_load", "m_mass",
             "m_fixed", "m_alive", "m_gen")}
    for k in ("s_m1", "s_m2", "s_m1gen", "s_m2gen", "s_rest", "s_k",
              "s_diam", "s_yield", "s_alive", "s_degen"):
        case[k] = getattr(st, "_" + k)[:s]
    for k in ("mode", "amp", "freq", "off", "per"):
        case["s_" + k] = getattr(st, "_s_act_" + k)[:s]
    planes, balls = engine.flatten_contacts(env)
    case.update(gravity=env.gravity.as_array(), drag=env.drag_coeff,
                planes=planes, balls=balls)
    return case


# ------------------------------------------------------------ cpu timing
def reference_case(args):
    """The workload as an oracle case, built by oracle/workloads.py (numpy
    only): the reference arm maps nothing from the product package
    (tests/test_workloads.py: same arrays as the product builder)."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import workloads
    return workloads.workload(args.config, args.n, args.robots)


def time_oracle(case, steps: int, warmup: int, threads: int,
                budget_s: float = 120.0):
    """Reference algorithm (oracle/ C restatement, fp64, slotted parallel =
    the reference's parallel+slotted backend) on the host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    sim = oracle.OracleSim(case, nthreads=threads)
    dt = 1e-4
    t = 0.0
    for _ in range(warmup):
        sim.step(t, dt, "slotted")
        t += dt
    done = 0
    w0 = time.perf_counter()
    while done < steps:
        sim.step(t, dt, "slotted")
        t += dt
        done += 1
        if time.perf_counter() - w0 > budget_s:
            break
    return done, time.perf_counter() - w0


# --------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region.

    NVML (nvidia_ml_py) polled every ~2 ms from a thread: the step call
    releases the GIL (ctypes), so the samples land inside the region even
    when it lasts only a few tens of ms.  Falls back to one nvidia-smi
    query after the region when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
               "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}

    def __init__(self, index: int, period_s: float = 0.002):
        import threading
        self.sm, self.mx, self.reasons = [], [], set()
        self.stop_evt = threading.Event()
        self.thread = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(
                self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return
        self.period = period_s
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def _sample(self):
        nv = self.nv
        self.sm.append(float(nv.nvmlDeviceGetClockInfo(self.h,
                                                       nv.NVML_CLOCK_SM)))
        self.mx.append(float(self.max_mhz))
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        for nm, b in self.REASONS.items():
            if bits & b:
                self.reasons.add(nm)

    def _run(self):
        while not self.stop_evt.is_set():
            try:
                self._sample()
            except Exception:
                return
            self.stop_evt.wait(self.period)

    def stop(self) -> dict | None:
        if self.thread is None:
            return self._smi_once()
        self.stop_evt.set()
        self.thread.join(timeout=5)
        if not self.sm:
            return self._smi_once()
        return {"sm_mhz": statistics.median(self.sm),
                "sm_max_mhz": max(self.mx), "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml, 2 ms"}

    @staticmethod
    def _smi_once():
        try:
            out = subprocess.run(
                ["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm",
                 "--format=csv,noheader,nounits"], capture_output=True,
                text=True, timeout=10).stdout.split(",")
            return {"sm_mhz": float(out[0]), "sm_max_mhz": float(out[1]),
                    "reasons": [], "samples": 1,
                    "source": "nvidia-smi after the region"}
        except Exception:
            return None


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def committed_traffic(workload_key: str):
    """dram bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(workload_key)
    except Exception:
        return None


# ------------------------------------------------------------------ main
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # one rank per GPU on the box; ranks beyond the device count (logic
        # tests with BENCH_DIST_BACKEND=gloo on one GPU) share devices
        from paper_1911_10274_b200 import _native
        local %= max(1, _native.device_count())
    dist = None
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    if world > 1:
        import torch
        import torch.distributed as dist
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        # nccl on the box (one rank per GPU); gloo lets the rank logic be
        # exercised with several ranks on one device
        dist.init_process_group(backend)

    def reduce_(x, op, dtype):
        import torch
        dev = f"cuda:{local}" if backend == "nccl" else "cpu"
        t = torch.tensor([x], device=dev, dtype=dtype)
        dist.all_reduce(t, op=op)
        return t.item()

    metric = "spring updates/sec"
    unit = "spring_updates/s"

    if args.impl == "reference":
        if rank != 0:
            return
        case = reference_case(args)
        workload = describe(args, 1)[0]
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle
        oracle.build()
        # all host threads (torchrun sets OMP_NUM_THREADS=1 per rank)
        threads = max(oracle.max_threads(), len(os.sched_getaffinity(0)))
        steps, wall = time_oracle(case, max(1, args.steps),
                                  max(1, args.warmup), threads,
                                  budget_s=180.0)
        springs = int(np.count_nonzero(case["s_alive"]))
        v = springs * steps / wall
        line = {"impl": "reference", "metric": metric, "value": v,
                "unit": unit, "n_gpus": args.gpus, "steps": steps,
                "warmup": args.warmup, "ms_per_step": 1e3 * wall /
                steps, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": v / PAPER_RATE, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload.replace(args.precision,
                                                        "fp64 (reference)"),
                           "masses": len(case["m_mass"]),
                           "springs": springs,
                           "inputs": "oracle/workloads.py (numpy; no "
                                     "product code on this arm)"},
                "cpu_baseline": {"value": v, "unit": unit, "cores": threads,
                                 "kind": "port",
                                 "sample": f"{steps} full steps of the "
                                           f"config-{args.config} workload, "
                                           f"oracle/ C restatement of "
                                           f"kernels.py, slotted, {threads} "
                                           f"threads"},
                "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if args.config == "E":
        return bench_config_e(args, rank, world, local, dist, reduce_)

    from paper_1911_10274_b200 import StepConfig, engine
    from paper_1911_10274_b200.control import SimController

    st, env, workload, scaling, extra = make_workload(args, rank, world)
    cfg = StepConfig(dt=1e-4, precision=args.precision, device=local,
                     accumulation=args.accumulation)
    springs, masses = st.spring_count, st.mass_count
    mir = engine.mirror_for(st, cfg)
    mir.push(st, env)
    acc = cfg.native_accumulation
    counters = np.zeros(3, np.int64)
    dt = cfg.dt
    step = 0

    def times(n):
        nonlocal step
        t = (step + np.arange(n, dtype=np.float64)) * dt
        step += n
        return t

    mir.ctx.step(times(max(3, args.warmup)), dt, acc, counters)  # warm-up
    st0 = mir.ctx.stats()
    launches0, fused0 = st0["kernel_launches"], st0["fused_launches"]
    if dist is not None:
        dist.barrier()
    mir.ctx.sync()
    clocks = ClockSampler(local)
    mir.ctx.timer_start()
    done, err = mir.ctx.step(times(args.steps), dt, acc, counters)
    call_ms = mir.ctx.timer_stop()
    # device time of the K step kernels: events on the library stream
    # right before the first and right after the last (sl_last_step_ms);
    # call_ms adds the call's status reset / read-back around them
    ms = mir.ctx.last_step_ms()
    clk = clocks.stop()
    stats = mir.ctx.stats()
    launches = stats["kernel_launches"] - launches0
    from paper_1911_10274_b200._native import STEP_PATHS
    kernel = (STEP_PATHS.get(stats["step_path"], "?")
              if args.accumulation == "gather" else "k_spring_atomic+k_mass")
    if stats["step_path"] == 4 and stats.get("split_batch"):
        kernel += f" (U={stats['split_batch']})"
    if stats.get("fused_launches", 0) > fused0:
        kernel = "k_fused_small (all steps in one launch)"
    if err:
        raise SystemExit(f"numerical abort at step {done}")
    sec = ms / 1e3
    if dist is not None:
        import torch
        sec = float(reduce_(sec, dist.ReduceOp.MAX, torch.float64))
        dist.barrier()
    total_springs = springs * world
    if dist is not None and args.config == "D":
        import torch
        total_springs = int(reduce_(springs, dist.ReduceOp.SUM, torch.int64))
    value = total_springs * args.steps / sec
    ms_per_step = 1e3 * sec / args.steps

    # fp64 parity mode (bit-exact with the reference) on the same workload:
    # the like-for-like (fp64 vs fp64) figure beside the reference arm
    fp64 = None
    if (args.config == "B" and args.precision != "fp64" and world == 1
            and not args.no_fp64):
        m64 = engine.DeviceMirror(local, "fp64")  # not the store's cache
        m64.push(st, env)
        c64 = np.zeros(3, np.int64)
        k64 = min(args.steps, 200)
        t64 = np.arange(max(3, args.warmup) + k64, dtype=np.float64) * dt
        m64.ctx.step(t64[:max(3, args.warmup)], dt, acc, c64)
        m64.ctx.sync()
        m64.ctx.step(t64[max(3, args.warmup):], dt, acc, c64)
        s64 = m64.ctx.last_step_ms() / 1e3
        st64 = m64.ctx.stats()
        fp64 = {"value": springs * k64 / s64, "unit": unit,
                "ms_per_step": 1e3 * s64 / k64, "steps": k64,
                "kernel": STEP_PATHS.get(st64["step_path"], "?"),
                "dtype": "f64",
                "parity": "bit-exact vs the reference (tests/"
                          "test_gpu_benchscale.py)"}
        m64.ctx.close()

    # roofline of the dominant kernel (the fused gather step: one launch per
    # step, so its average duration is the per-step device time)
    algo = algorithmic_bytes(springs, masses, args.precision, extra)
    peak, peak_kind = peak_hbm()
    achieved = algo / (sec / args.steps) / 1e9
    key = (f"{args.n}^3/{args.precision}/{args.accumulation}"
           if args.config == "B" else
           f"{args.config}{args.robots if args.config == 'D' else ''}/"
           f"{args.precision}/{args.accumulation}")
    traffic = committed_traffic(key)
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak,
            "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
            "peak_kind": peak_kind, "algorithmic_bytes_per_step": algo,
            "bytes_per_spring_update": algo / springs,
            "kernel": kernel}
    if traffic:
        # DRAM bytes the kernel really moves (committed ncu capture) at the
        # measured step time: below `achieved` when the layout compresses
        # the algorithmic stream (window kernel: material table, 16-bit
        # window indices)
        roof["traffic_gbs"] = traffic / (sec / args.steps) / 1e9
        roof["traffic_frac"] = roof["traffic_gbs"] / peak

    # e2e through the public API, host store authoritative at both ends: an
    # RL / control segment in steady state -- set-state (the inputs: new
    # positions and velocities written into the host store, io.apply_
    # snapshot), run K steps (SimController.start -> wait_for_event), get-
    # state (snapshot).  Untimed segments first bring host and device in
    # sync, as a running controller is between segments; the timed one
    # then moves the columns the host touched (pos, vel) up and the state
    # down (DeviceMirror.push / pull).
    e2e = None
    if not args.no_e2e:
        from paper_1911_10274_b200 import io as sio
        ctl = SimController(st, env, cfg)
        k = args.steps
        m = st.mass_slot_count
        for _ in range(E2E_WARM):  # untimed segments: steady state (pools warm)
            ctl.start(k * dt)
            ctl.wait_for_event()
            warm = ctl.snapshot()
        ids = warm.ids.copy()
        pos_in = _native_pinned_copy(warm.positions)
        vel_in = _native_pinned_copy(warm.velocities)
        del warm
        full0 = getattr(engine.mirror_for(st, cfg), "full_pushes", 0)
        # E2E_REPS timed segments (each: set-state, K steps, get-state) and
        # their median: one ~5 ms segment is at the mercy of host noise
        walls = []
        for _ in range(E2E_REPS):
            if dist is not None:
                dist.barrier()
            w0 = time.perf_counter()
            sio.apply_snapshot(st, ids, pos_in, vel_in)
            ctl.start(k * dt)
            rep = ctl.wait_for_event()
            snap = ctl.snapshot()
            walls.append(time.perf_counter() - w0)
            del snap
        snap_rows = m
        wall = float(np.median(walls))
        full = getattr(engine.mirror_for(st, cfg), "full_pushes", 0) - full0
        ctl.stop()
        assert rep.step_count == (E2E_WARM + E2E_REPS) * k, rep
        if dist is not None:
            import torch
            wall = float(reduce_(wall, dist.ReduceOp.MAX, torch.float64))
        h2d = m * 48 if not full else m * (5 * 24 + 8 + 1 + 1 + 8)
        # the pause moves the snapshot's positions / velocities; the store's
        # state columns stay on the device until the host reads them
        # (engine._DeferredPull) -- nothing reads them in this segment
        d2h = m * 2 * 24
        e2e = {"value": world * springs * k / wall, "unit": unit,
               "h2d_bytes_per_step": h2d / k, "d2h_bytes_per_step": d2h / k,
               "wall_s": wall, "api": "io.apply_snapshot + SimController."
                                      "start/wait_for_event/snapshot",
               "segment": "set-state, K steps, get-state (steady state)",
               "segments": E2E_REPS, "aggregate": "median wall per segment",
               "segment_walls_s": [round(w, 6) for w in walls],
               "snapshot_rows": int(snap_rows)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            sys.path.insert(0, os.path.join(ROOT, "oracle"))
            import oracle
            oracle.build()
            thr = max(oracle.max_threads(), len(os.sched_getaffinity(0)))
            case2 = reference_case(args)
            n_s, wall = time_oracle(case2, 3, 1, thr, budget_s=30.0)
            cpu = {"value": int(case2["s_alive"].sum()) * n_s / wall,
                   "unit": unit,
                   "cores": thr, "kind": "port",
                   "sample": f"{n_s} steps of the same config-"
                             f"{args.config} workload (fp64, slotted, "
                             f"oracle/ C restatement of kernels.py, OpenMP "
                             f"{thr} threads)"}
        except Exception as exc:  # baseline is reported, never fatal
            cpu = {"error": str(exc)}

    if rank == 0:
        line = {"metric": metric, "value": value, "unit": unit,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": scaling, "vs_baseline": value / PAPER_RATE,
                "dtype": "f32" if args.precision == "fp32" else "f64",
                "data": "synthetic",
                "config": {"workload": workload, "masses": masses,
                           "springs": springs,
                           "total_springs": total_springs,
                           "per_gpu_instances": (
                               "robot shard" if args.config == "D" else 1),
                           "precision": args.precision,
                           "precision_detail": {
                               "fp32": "fp32 arithmetic; positions "
                                       "compensated (fp32 + fp32 low part)",
                               "mixed": "fp64 state and force arithmetic, "
                                        "fp32 (k, L0) storage",
                               "fp64": "fp64, bit-exact with the reference"
                           }[args.precision],
                           "accumulation": args.accumulation,
                           "l2": ("working set > 126 MB L2 every step "
                                  "(no flush needed)" if args.config == "B"
                                  and args.n >= 100 else
                                  "working set fits L2 (small bodies / "
                                  "shards); no flush: an L2-resident "
                                  "simulation is the workload"),
                           "parallelism": f"batched instances x{world}"},
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clk,
                "call_ms_per_step": call_ms / args.steps,
                "fp64_parity_mode": fp64,
                "vs_baseline_ref": "PAPER.md:10 3.0e8 spring updates/s"}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def bench_config_e(args, rank, world, local, dist, reduce_):
    """Config E: one lattice partitioned by mass
    range over the ranks; each rank steps its x-slab (owned masses +
    ghosts), the halo rides on the step kernels (distributed.HaloRun).
    value = all springs x K / max over ranks of the step-kernel time."""
    import torch
    from paper_1911_10274_b200 import _native
    from paper_1911_10274_b200.distributed import HaloRun
    from paper_1911_10274_b200.partition import (even_cuts, halo_plans,
                                                 partition_case)
    metric, unit = "spring updates/sec", "spring_updates/s"
    n = args.n
    st, env = build_workload(n)
    case = store_case(st, env)
    case.update(gc_kind=np.zeros(0, np.int8), gc_vec=np.zeros((0, 3)))
    springs = st.spring_count
    cuts = even_cuts(st.mass_count, world, align=n * n)
    shards = partition_case(case, cuts, ranks=[rank])
    plans = halo_plans(shards)
    run = HaloRun(shards[rank], plans, local, args.precision)
    if world > 1:
        run.connect_ipc()
    acc = _native.ACC_GATHER if args.accumulation == "gather" else \
        _native.ACC_ATOMIC
    dt = 1e-4
    warm = max(3, args.warmup)
    times = np.arange(warm + args.steps, dtype=np.float64) * dt
    run.step(times[:warm], dt, acc)
    if dist is not None:
        dist.barrier()
    run.ctx.sync()
    clocks = ClockSampler(local)
    run.ctx.timer_start()
    done, err = run.step(times[warm:], dt, acc)
    call_ms = run.ctx.timer_stop()
    ms = run.ctx.last_step_ms()
    clk = clocks.stop()
    if err:
        raise SystemExit(f"numerical abort at step {done}")
    sec = ms / 1e3
    if dist is not None:
        sec = float(reduce_(sec, dist.ReduceOp.MAX, torch.float64))
    value = springs * args.steps / sec
    local_springs = len(shards[rank].spring_slots)
    algo = algorithmic_bytes(springs, st.mass_count, args.precision)
    peak, peak_kind = peak_hbm()
    stats = run.ctx.stats()
    # e2e through the same API with host buffers: this rank's state up,
    # K steps, its owned state down
    # (a control segment as config B's: new positions / velocities up from
    # page-locked host buffers, K steps, positions / velocities down into
    # page-locked buffers; median of E2E_REPS segments)
    m_loc = len(shards[rank].local_to_global)
    c = shards[rank].case
    pin = [_native.pinned_empty((m_loc, 3), np.float64) for _ in range(4)]
    pin[0][...] = np.asarray(c["m_pos"]).reshape(m_loc, 3)
    pin[1][...] = np.asarray(c["m_vel"]).reshape(m_loc, 3)
    walls = []
    for _ in range(E2E_REPS):
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        run.ctx.write_state(pin[0], pin[1], None)
        if world > 1:
            dist.barrier()
        run.step(times[warm:], dt, acc)
        run.ctx.download_masses(pin[2], pin[3])
        walls.append(time.perf_counter() - w0)
    wall = float(np.median(walls))
    if dist is not None:
        wall = float(reduce_(wall, dist.ReduceOp.MAX, torch.float64))
    run.close()
    if rank == 0:
        line = {"metric": metric, "value": value, "unit": unit,
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": 1e3 * sec / args.steps,
                "higher_is_better": True, "scaling": "strong",
                "vs_baseline": value / PAPER_RATE,
                "dtype": "f32" if args.precision == "fp32" else "f64",
                "data": "synthetic",
                "config": {"workload": describe(args, world)[0],
                           "masses": st.mass_count, "springs": springs,
                           "rank0_springs_incl_cross": local_springs,
                           "precision": args.precision,
                           "accumulation": args.accumulation,
                           "parallelism": f"x-slab partition x{world}",
                           "l2": "working set > L2 every step"},
                "roofline": {"bound": "hbm", "achieved":
                             algo / world / (sec / args.steps) / 1e9,
                             "peak": peak, "unit": "GB/s",
                             "frac": algo / world / (sec / args.steps) / 1e9
                             / peak, "traffic": None, "peak_kind": peak_kind,
                             "algorithmic_bytes_per_step_per_gpu":
                                 algo / world,
                             "kernel": _native.STEP_PATHS.get(
                                 stats["step_path"], "?") +
                             (" + k_halo_sync" if world > 1 else "")},
                "e2e": {"value": springs * args.steps / wall, "unit": unit,
                        "h2d_bytes_per_step": m_loc * 48 / args.steps,
                        "d2h_bytes_per_step": m_loc * 48 / args.steps,
                        "segments": E2E_REPS,
                        "segment_walls_s": [round(w, 6) for w in walls],
                        "api": "sl_write_state + sl_step + "
                               "sl_download_masses per rank"},
                "gpu_launches": args.steps * (2 if world > 1 else 1),
                "call_ms_per_step": call_ms / args.steps,
                "clocks": clk, "cpu_baseline": None}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
