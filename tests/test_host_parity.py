"""Host side (store, builder, actuation, constraint flattening) vs the
reference, on CPU.

Every golden case in tests/golden was built by the REFERENCE's own builder /
store / actuation API (tests/golden/make_golden.py).  Rebuilding the same
cases with this package's mirror of that API must give the identical input
arrays -- slot order, generations, rest lengths, stiffnesses, masses,
actuation parameters, constraint CSR -- bit for bit: that is where
"connectivity and indexing bit-exact" (north_star) starts, before any
kernel runs.
"""
import numpy as np
import pytest

from conftest import load_golden
from paper_1911_10274_b200 import (ActuationParams, ContactBall,
                                   ContactPlane, Environment,
                                   LocalConstraint, Mass, Material,
                                   ObjectStore, Spring, Vec3, engine)
from paper_1911_10274_b200.actuation import configure_worm
from paper_1911_10274_b200.builder import (LatticeSpec, build_lattice,
                                           grid_springs,
                                           lattice_spring_count)


def our_case(st: ObjectStore, env: Environment) -> dict:
    m, s = st.mass_slot_count, st.spring_slot_count
    planes, balls = engine.flatten_contacts(env)
    gk, gv = engine.global_constraint_arrays(st)
    lc_off, lc_kind, lc_vec = engine.local_constraint_csr(st)
    return {
        "m_pos": st._m_pos[:m], "m_vel": st._m_vel[:m],
        "m_acc": st._m_acc[:m], "m_fext": st._m_fext[:m],
        "m_load": st._m_load[:m], "m_mass": st._m_mass[:m],
        "m_fixed": st._m_fixed[:m].astype(np.uint8),
        "m_alive": st._m_alive[:m].astype(np.uint8), "m_gen": st._m_gen[:m],
        "s_m1": st._s_m1[:s], "s_m2": st._s_m2[:s],
        "s_m1gen": st._s_m1gen[:s], "s_m2gen": st._s_m2gen[:s],
        "s_rest": st._s_rest[:s], "s_k": st._s_k[:s],
        "s_diam": st._s_diam[:s], "s_yield": st._s_yield[:s],
        "s_mode": st._s_act_mode[:s], "s_amp": st._s_act_amp[:s],
        "s_freq": st._s_act_freq[:s], "s_off": st._s_act_off[:s],
        "s_per": st._s_act_per[:s],
        "s_alive": st._s_alive[:s].astype(np.uint8),
        "s_degen": st._s_degen[:s].astype(np.uint8),
        "gravity": env.gravity.as_array(), "drag": np.float64(env.drag_coeff),
        "planes": planes, "balls": balls, "gc_kind": gk, "gc_vec": gv,
        "lc_off": lc_off, "lc_kind": lc_kind, "lc_vec": lc_vec,
    }


# --- the case factories of tests/golden/make_golden.py, on this package ---
def lattice(n, spacing=0.05, mat=None, corner=(0, 0, 0), stretch=None,
            nxyz=None, diameter=1e-3):
    mat = mat or Material(elastic_modulus=1e5, density=1000.0)
    st = ObjectStore()
    nx, ny, nz = nxyz or (n, n, n)
    body = build_lattice(LatticeSpec(corner=Vec3(*corner), nx=nx, ny=ny,
                                     nz=nz, spacing=spacing, material=mat,
                                     diameter=diameter), st)
    if stretch:
        st._m_pos[body.mass_handles.slots] *= stretch
    return st, body


def ground(k, mu_s, mu_k, offset=0.0):
    return ContactPlane(normal=Vec3(0, 0, 1), offset=offset, stiffness=k,
                        static_friction=mu_s, kinetic_friction=mu_k)


CUBE = Material(elastic_modulus=1e6, density=1000.0)
G = Vec3(0, 0, -9.81)


def case_cube10_drop():
    return (lattice(10, 0.1, CUBE, corner=(0, 0, 0.3))[0],
            Environment(gravity=G, contacts=[ground(2000.0, 1.0, 0.8)]))


def case_cube10_contact():
    return (lattice(10, 0.1, CUBE, corner=(0, 0, -0.002), stretch=1.01)[0],
            Environment(gravity=G, contacts=[ground(2000.0, 1.0, 0.8)]))


def case_lat3_contact_drag():
    return (lattice(3, corner=(0, 0, 0.01), stretch=1.05)[0],
            Environment(gravity=G, drag_coeff=0.01,
                        contacts=[ground(500.0, 0.6, 0.5)]))


def case_worm():
    st, body = lattice(0, 0.05, CUBE, nxyz=(20, 6, 6))
    configure_worm(body, st)
    return st, Environment(gravity=G, drag_coeff=0.01,
                           contacts=[ground(500.0, 1.0, 0.8)])


def case_actuated_quiescent():
    st, body = lattice(4, stretch=1.02)
    for i, h in enumerate(body.spring_handles):
        st.set_spring_field(h, "actuation", ActuationParams(
            amplitude=0.3, frequency=50.0, offset=1e-3 * (i % 7),
            period=0.013, quiescent_before_offset=bool(i % 2)))
    return st, Environment(gravity=G)


def case_yield_break():
    nylon = Material(elastic_modulus=4.56e9, density=1150.0,
                     yield_stress=8e7)
    st, body = lattice(4, spacing=0.01, mat=nylon, stretch=1.0)
    slots = body.mass_handles.slots
    x = st._m_pos[slots, 0]
    st._m_pos[slots, 0] = x * (1.0 + 0.05 * (x > 0.015))
    return st, Environment(gravity=Vec3(0, 0, 0))


def case_constraints_contacts():
    st, body = lattice(4, stretch=1.03, corner=(0.0, 0.0, 0.02))
    hs = list(body.mass_handles)
    st.set_mass_field(hs[0], "fixed", True)
    st.set_mass_field(hs[5], "fixed", True)
    st.set_mass_field(hs[7], "local_constraints",
                      (LocalConstraint.direction((1, 1, 0)),))
    st.set_mass_field(hs[9], "local_constraints",
                      (LocalConstraint.plane((0, 0, 1)),
                       LocalConstraint.direction((1, 0, 0))))
    st.set_applied_load(hs[20], Vec3(0.3, -0.2, 0.5))
    st.set_mass_field(hs[33], "f_ext", Vec3(1.0, 2.0, 3.0))
    st.add_global_constraint(LocalConstraint.plane((0, 1, 0)))
    env = Environment(gravity=G, drag_coeff=0.05, contacts=[
        ground(800.0, 0.7, 0.4),
        ContactPlane(normal=Vec3(1, 0, 0), offset=0.01, stiffness=300.0,
                     static_friction=0.2, kinetic_friction=0.1),
        ContactBall(center=Vec3(0.08, 0.08, 0.2), radius=0.12,
                    stiffness=400.0)])
    return st, env


def case_topology_edits():
    st, body = lattice(4, stretch=1.04)
    hs = list(body.mass_handles)
    sh = list(body.spring_handles)
    st.delete_mass(hs[6])
    st.delete_mass(hs[21])
    for i in (3, 40, 41, 100):
        st.delete_spring(sh[i])
    a = st.create_mass(Mass(pos=Vec3(0.3, 0.3, 0.3), m=0.01))
    b = st.create_mass(Mass(pos=Vec3(0.3, 0.3, 0.3), m=0.01))
    st.create_spring(Spring(m1=a, m2=b, rest_length=0.05, stiffness=5.0))
    st.create_spring(Spring(m1=hs[1], m2=a, rest_length=0.2, stiffness=7.0))
    st.create_spring(Spring(m1=b, m2=hs[60], rest_length=0.2, stiffness=7.0,
                            diameter=1e-3, yield_stress=1e3))
    return st, Environment(gravity=G)


def case_nan_abort():
    st = ObjectStore()
    a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
    b = st.create_mass(Mass(pos=Vec3(1, 0, 0), m=1e-30))
    st.create_spring(Spring(m1=a, m2=b, rest_length=0.1, stiffness=1e30))
    return st, Environment(gravity=Vec3(0, 0, 0))


FACTORIES = {name[5:]: fn for name, fn in globals().items()
             if name.startswith("case_")}


@pytest.mark.parametrize("name", sorted(FACTORIES))
def test_inputs_match_reference_bitwise(name):
    st, env = FACTORIES[name]()
    ours = our_case(st, env)
    ref = load_golden(name)
    for key, val in ours.items():
        want = ref[key]
        got = np.asarray(val)
        if key in ("gc_vec", "lc_vec", "planes", "balls"):
            want = want.reshape(-1, got.shape[-1] if got.ndim > 1 else 1)
            got = got.reshape(want.shape)
        assert got.shape == want.shape, (key, got.shape, want.shape)
        assert got.astype(want.dtype).tobytes() == want.tobytes(), key


@pytest.mark.parametrize("n", [(1, 1, 1), (2, 3, 4), (5, 5, 5), (7, 2, 9)])
def test_lattice_counts_and_connectivity(n):
    """Count formula (builder.py:132-138) and brute-force same-cell pairs
    (tests/oracle.py:151-170 analogue)."""
    nx, ny, nz = n
    a, b = grid_springs(nx, ny, nz)
    assert len(a) == lattice_spring_count(nx, ny, nz)
    idx = np.indices((nx, ny, nz)).reshape(3, -1).T
    want = set()
    for p in range(len(idx)):
        for q in range(p + 1, len(idx)):
            d = np.abs(idx[p] - idx[q])
            if d.max() == 1:
                want.add((p, q))
    got = {(min(x, y), max(x, y)) for x, y in zip(a.tolist(), b.tolist())}
    assert got == want and len(got) == len(a)


def test_stiffness_max_tracker_exact_through_edits():
    """ObjectStore keeps the largest alive stiffness exact through creates,
    deletes and retunes (engine.check_stability's k_max without an O(S)
    scan per edit): equal to the brute-force masked max at every step."""
    import numpy as np
    from paper_1911_10274_b200 import (Mass, ObjectStore, Spring, Vec3,
                                       engine)
    rng = np.random.default_rng(5)
    st = ObjectStore()
    ms = [st.create_mass(Mass(pos=Vec3(float(i), 0.0, 0.0), m=1.0))
          for i in range(40)]
    springs = []
    for step in range(300):
        op = rng.integers(0, 3)
        if op == 0 or not springs:
            a, b = rng.choice(40, 2, replace=False)
            k = float(rng.choice([5.0, 7.0, 9.0, float(rng.uniform(0, 10))]))
            springs.append(st.create_spring(Spring(
                m1=ms[a], m2=ms[b], rest_length=1.0, stiffness=k)))
        elif op == 1:
            st.delete_spring(springs.pop(int(rng.integers(len(springs)))))
        else:
            h = springs[int(rng.integers(len(springs)))]
            st.set_spring_field(h, "stiffness",
                                float(rng.choice([9.0, float(rng.uniform(0, 10))])))
        s = st.spring_slot_count
        alive = st._s_alive[:s].astype(bool)
        want = float(st._s_k[:s][alive].max()) if alive.any() else None
        t = st.__dict__.get("_kmax_track")
        if t is not None and want is not None:
            assert t[0] == want, (step, t, want)
        # the stability ratio uses the same k_max as a fresh scan
        r = engine.check_stability(st, 1e-3)
        if want is not None:
            assert abs(r - 1e-3 * (want / 1.0) ** 0.5) < 1e-15
