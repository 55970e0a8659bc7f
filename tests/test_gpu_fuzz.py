"""Randomised unstructured meshes through every production path, against
the reference oracle (oracle/, pinned to the reference's own trajectories).

Each seed builds a random store-format case: masses scattered in a box
(some fixed, some dead, random generations), springs between x-sorted
neighbours (banded: the window kernel), plus random long-range springs
(wide windows: the split / gather fallbacks) or many small components (the
fused multi-step kernel), duplicate pairs, a zero-length spring, stale
generation endpoints (killed as invalid), breakable springs, sine
actuation, ground and inclined planes, a ball, global and local
constraints.

* fp64: positions, velocities, spring flags and counters bit-identical to
  the reference (unactuated cases; contact, friction, yield breaks and
  constraints active).
* fp32 / mixed: within 1e-4 (positions) of the fp64 reference over 30
  steps with no contact and no breakable springs (threshold decisions are
  discontinuous), actuation on; connectivity bit-exact.
"""
import numpy as np
import pytest

import oracle as orc
from conftest import case_context, rel_maxnorm

pytestmark = pytest.mark.gpu


def rand_case(seed, shape, contact, actuated, yields, zero_length=True):
    rng = np.random.default_rng(seed)
    m = int(rng.integers(300, 2200))
    pos = rng.uniform(-1.0, 1.0, (m, 3))
    pos[:, 2] = rng.uniform(-0.01 if contact else 0.3, 1.0, m)
    vel = rng.normal(0.0, 0.05, (m, 3))
    mass = rng.uniform(0.05, 2.0, m)
    fixed = rng.random(m) < 0.03
    alive = rng.random(m) > 0.02
    gen = rng.integers(0, 3, m).astype(np.int64)
    order = np.argsort(pos[:, 0], kind="stable")
    a_l, b_l = [], []
    if shape == "components":  # bodies: disjoint contiguous slot ranges
        i = 0
        while i < m:
            g = int(rng.integers(10, 60))
            idx = np.arange(i, min(i + g, m))
            for off in range(1, 5):
                a_l.append(idx[:-off])
                b_l.append(idx[off:])
            perm = rng.permutation(idx)  # plus random pairs inside the body
            a_l.append(perm[:len(perm) // 2])
            b_l.append(perm[len(perm) - len(perm) // 2:][:len(perm) // 2])
            i += g
    else:
        for off in range(1, 7):
            a_l.append(order[:-off])
            b_l.append(order[off:])
    a = np.concatenate(a_l)
    b = np.concatenate(b_l)
    if shape == "longrange":
        extra = m // 2
        a = np.concatenate([a, rng.integers(0, m, extra)])
        b = np.concatenate([b, rng.integers(0, m, extra)])
    keep = a != b
    a, b = a[keep], b[keep]
    dup = rng.integers(0, len(a), 5)  # duplicate pairs
    a, b = np.concatenate([a, b[dup]]), np.concatenate([b, a[dup]])
    flip = rng.random(len(a)) < 0.5
    a, b = np.where(flip, b, a), np.where(flip, a, b)
    s = len(a)
    # one zero-length spring (coincident endpoints)
    z = int(rng.integers(0, s))
    if zero_length:
        pos[b[z]] = pos[a[z]]
    d = np.linalg.norm(pos[b] - pos[a], axis=1)
    rest = np.where(d > 0, d * rng.uniform(0.9, 1.1, s), 0.05)
    k = rng.uniform(10.0, 400.0, s)
    if shape == "components":
        # a few materials (the fused kernel keeps <= 64 (k, L0) pairs per
        # group, as builder bodies have): quantised rest lengths, soft k
        rest = rng.choice([0.5, 1.0, 1.5], s)
        k = rng.choice([2.0, 5.0, 10.0], s)
    m1gen, m2gen = gen[a].copy(), gen[b].copy()
    stale = rng.random(s) < 0.01
    m1gen[stale] += 1
    diam = rng.uniform(1e-3, 3e-3, s)
    ys = np.full(s, np.inf)
    if yields:  # some springs break within the run, most never do
        weak = rng.random(s) < 0.05
        area = 0.25 * np.pi * diam * diam
        ys[weak] = np.abs(k[weak] * (d[weak] - rest[weak])) / area[weak] \
            * rng.uniform(0.3, 3.0, int(weak.sum())) + 1.0
    mode = np.zeros(s, np.int8)
    amp, freq = np.zeros(s), np.zeros(s)
    off, per = np.zeros(s), np.ones(s)
    if actuated:
        r = rng.random(s)
        mode[r < 0.1] = 1
        mode[(r >= 0.1) & (r < 0.15)] = 2
        act = mode > 0
        amp[act] = rng.uniform(0.05, 0.2, int(act.sum()))
        freq[act] = rng.uniform(5.0, 30.0, int(act.sum()))
        off[act] = rng.uniform(0.0, 0.5, int(act.sum()))
        per[act] = rng.uniform(0.5, 1.5, int(act.sum()))
        if shape == "components":  # worm-like: a few waveforms
            na = int(act.sum())
            amp[act] = 0.1
            freq[act] = 20.0
            off[act] = rng.choice([0.0, 0.1], na)
            per[act] = 1.0
    s_alive = rng.random(s) > 0.03
    planes = np.zeros((0, 7))
    balls = np.zeros((0, 5))
    if contact:
        n2 = np.array([0.3, 0.0, 1.0]) / np.linalg.norm([0.3, 0.0, 1.0])
        planes = np.array([[0, 0, 1, 0.0, 2000.0, 1.0, 0.8],
                           [*n2, -0.2, 1500.0, 0.6, 0.4]])
        balls = np.array([[0.2, -0.3, 0.1, 0.25, 800.0]])
    gk = rng.integers(0, 3)
    gc_kind = np.array([1], np.int8) if gk == 1 else np.zeros(0, np.int8)
    gc_vec = np.array([[0.0, 1.0, 0.0]]) if gk == 1 else np.zeros((0, 3))
    lc_n = np.zeros(m, np.int64)
    lc_n[rng.random(m) < 0.02] = 1
    lc_off = np.zeros(m + 1, np.int64)
    lc_off[1:] = np.cumsum(lc_n)
    L = int(lc_off[-1])
    lc_kind = rng.integers(0, 2, L).astype(np.int8)
    lc_vec = rng.normal(size=(L, 3))
    lc_vec /= np.linalg.norm(lc_vec, axis=1, keepdims=True)
    return dict(m_pos=pos, m_vel=vel, m_acc=np.zeros((m, 3)),
                m_fext=np.zeros((m, 3)), m_load=rng.normal(0, 0.01, (m, 3)),
                m_mass=mass, m_fixed=fixed, m_alive=alive, m_gen=gen,
                s_m1=a.astype(np.int64), s_m2=b.astype(np.int64),
                s_m1gen=m1gen, s_m2gen=m2gen, s_rest=rest, s_k=k,
                s_diam=diam, s_yield=ys, s_alive=s_alive,
                s_degen=np.zeros(s, bool), s_mode=mode, s_amp=amp,
                s_freq=freq, s_off=off, s_per=per,
                gravity=np.array([0.0, 0.0, -9.81]), drag=0.05,
                planes=planes, balls=balls, gc_kind=gc_kind, gc_vec=gc_vec,
                lc_off=lc_off, lc_kind=lc_kind, lc_vec=lc_vec)


def run(case, precision, n, dt=1e-4):
    ctx = case_context(case, precision)
    c = np.zeros(3, np.int64)
    times = np.arange(n, dtype=np.float64) * dt
    done, err = ctx.step(times, dt, 0, c)
    assert err == 0 and done == n
    st = ctx.stats()
    m, s = len(case["m_mass"]), len(case["s_m1"])
    pos, vel = np.zeros((m, 3)), np.zeros((m, 3))
    ctx.download_masses(pos, vel)
    alive, degen = np.zeros(s, np.uint8), np.zeros(s, np.uint8)
    ctx.download_springs(alive, degen)
    ctx.close()
    ref = orc.OracleSim(case)
    for k in range(n):
        assert ref.step(float(times[k]), dt) == 0
    return (pos, vel, alive.astype(bool), degen.astype(bool), c, st,
            ref.c, ref.counters)


@pytest.mark.parametrize("shape", ["banded", "longrange", "components"])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_fuzz_fp64_bit_exact(seed, shape):
    case = rand_case(100 * seed + 7, shape, contact=True, actuated=False,
                     yields=True)
    pos, vel, alive, degen, c, st, ref, rc = run(case, "fp64", 40)
    assert pos.tobytes() == ref["m_pos"].tobytes()
    assert vel.tobytes() == ref["m_vel"].tobytes()
    assert np.array_equal(alive, ref["s_alive"])
    assert np.array_equal(degen, ref["s_degen"])
    assert c.tolist() == rc.tolist()


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
@pytest.mark.parametrize("shape", ["banded", "longrange", "components"])
@pytest.mark.parametrize("seed", [0, 1])
def test_fuzz_tolerance_modes(seed, shape, precision):
    # the components case without a zero-length spring: the fused kernel
    # takes contexts with no special (exact-path) masses
    case = rand_case(100 * seed + 11, shape, contact=False, actuated=True,
                     yields=False, zero_length=shape != "components")
    pos, vel, alive, degen, c, st, ref, rc = run(case, precision, 30)
    assert rel_maxnorm(pos, ref["m_pos"]) < 1e-4
    assert rel_maxnorm(vel, ref["m_vel"]) < 1e-4
    assert np.array_equal(alive, ref["s_alive"])
    assert np.array_equal(degen, ref["s_degen"])
    assert c.tolist() == rc.tolist()
    if precision == "fp32" and shape == "components":
        assert st["fused_launches"] > 0
