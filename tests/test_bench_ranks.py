"""bench.py's multi-rank logic on CPU (no GPU): config D shards tile the
global robot swarm exactly (each rank a contiguous body range, the union
equals the single-rank build), and the reference arm under torchrun with
two gloo ranks prints exactly one JSON line from rank 0."""
import argparse
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _args(**kw):
    a = argparse.Namespace(config="D", robots=10, n=4, precision="fp32",
                           accumulation="gather")
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("world", [1, 2, 3, 4])
def test_config_d_shards_tile_the_swarm(world):
    whole, _, _, _, _ = bench.make_workload(_args(), 0, 1)
    pos, springs = [], 0
    for rank in range(world):
        st, _, desc, scaling, extra = bench.make_workload(_args(), rank, world)
        assert extra == 1 and f"over {world} rank" in desc
        assert scaling == ("strong" if world > 1 else "weak")
        pos.append(st._m_pos[:st.mass_slot_count])
        springs += st.spring_count
    assert springs == whole.spring_count
    got = np.concatenate(pos)
    assert got.tobytes() == whole._m_pos[:whole.mass_slot_count].tobytes()


def test_reference_arm_two_gloo_ranks_one_line():
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=2", "--master-addr=127.0.0.1",
           "--master-port=29531", "bench.py", "--impl", "reference",
           "--gpus", "2", "--edge", "6", "--steps", "2", "--warmup", "1"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
    assert d["e2e"]["h2d_bytes_per_step"] == 0


def test_config_a_is_the_reference_bouncing_cube():
    """bench --config A builds scenarios/bouncing_cube.ini's cube: 10^3
    masses, 10,476 springs, corner at z = 0.3."""
    st, env, desc, scaling, extra = bench.make_workload(_args(config="A"),
                                                        0, 1)
    assert st.mass_count == 1000 and st.spring_count == 10476
    assert float(st._m_pos[:1000, 2].min()) == 0.3 and extra == 0
    assert desc.startswith("A: 10^3 bouncing cube") and scaling == "weak"
    assert len(env.contacts) == 1
