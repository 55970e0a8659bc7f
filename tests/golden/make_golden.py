"""Generate golden trajectories by running the REFERENCE itself.

Run in the build container only (needs /root/reference and numba):

    python tests/golden/make_golden.py

It imports ``softlat`` from /root/reference/pkg/src, builds each case with the
reference's own builder / store / actuation API, snapshots the store arrays
(the inputs), steps with the reference's serial backend
(``engine.step`` -> kernels.spring_linear_serial + kernels.mass_pass_serial,
engine.py:158-264) and records the outputs.  It also asserts the reference's
serial-slotted backend agrees bitwise (engine.py:105-118), which is the
accumulation order our deterministic gather variant reproduces.

Nothing on the GPU box reads /root/reference: the committed *.npz files are
the only artefacts the tests use.
"""
from __future__ import annotations

import math
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

os.environ.setdefault("NUMBA_CACHE_DIR",
                      os.path.join(tempfile.gettempdir(), "softlat_numba"))
sys.path.insert(0, REF)

from softlat import (ContactBall, ContactPlane, Environment,  # noqa: E402
                     LocalConstraint, Mass, Material, Spring, StepConfig,
                     Vec3, engine)
from softlat.actuation import ActuationParams, configure_worm  # noqa: E402
from softlat.builder import LatticeSpec, build_lattice  # noqa: E402
from softlat.store import ObjectStore  # noqa: E402


def store_case(st: ObjectStore, env: Environment) -> dict:
    """Flatten a reference store + environment exactly as engine.py does."""
    m, s = st.mass_slot_count, st.spring_slot_count
    engine._refresh_constraints(st, engine._cache_for(st))
    cache = engine._cache_for(st)
    planes = np.zeros((len(env.planes()), 7))
    for p, pl in enumerate(env.planes()):
        planes[p] = [*pl.normal.as_tuple(), pl.offset, pl.stiffness,
                     pl.static_friction, pl.kinetic_friction]
    balls = np.zeros((len(env.balls()), 5))
    for b, bl in enumerate(env.balls()):
        balls[b] = [*bl.center.as_tuple(), bl.radius, bl.stiffness]
    return {
        "m_pos": st._m_pos[:m].copy(), "m_vel": st._m_vel[:m].copy(),
        "m_acc": st._m_acc[:m].copy(), "m_fext": st._m_fext[:m].copy(),
        "m_load": st._m_load[:m].copy(), "m_mass": st._m_mass[:m].copy(),
        "m_fixed": st._m_fixed[:m].astype(np.uint8),
        "m_alive": st._m_alive[:m].astype(np.uint8),
        "m_gen": st._m_gen[:m].copy(),
        "s_m1": st._s_m1[:s].copy(), "s_m2": st._s_m2[:s].copy(),
        "s_m1gen": st._s_m1gen[:s].copy(), "s_m2gen": st._s_m2gen[:s].copy(),
        "s_rest": st._s_rest[:s].copy(), "s_k": st._s_k[:s].copy(),
        "s_diam": st._s_diam[:s].copy(), "s_yield": st._s_yield[:s].copy(),
        "s_mode": st._s_act_mode[:s].copy(), "s_amp": st._s_act_amp[:s].copy(),
        "s_freq": st._s_act_freq[:s].copy(), "s_off": st._s_act_off[:s].copy(),
        "s_per": st._s_act_per[:s].copy(),
        "s_alive": st._s_alive[:s].astype(np.uint8),
        "s_degen": st._s_degen[:s].astype(np.uint8),
        "gravity": np.array(env.gravity.as_tuple()),
        "drag": np.float64(env.drag_coeff), "planes": planes, "balls": balls,
        "gc_kind": cache.gc_kind.copy(), "gc_vec": cache.gc_vec.reshape(-1, 3),
        "lc_off": cache.lc_off.copy(), "lc_kind": cache.lc_kind.copy(),
        "lc_vec": cache.lc_vec.reshape(-1, 3),
    }


def run_reference(st, env, dt, steps, checkpoints, time_rule, out, tag="",
                  accumulation="linearizable"):
    cfg = StepConfig(dt=dt, accumulation=accumulation)
    t = 0.0
    counters = np.zeros(3, np.int64)
    done = 0
    err = 0
    for n in range(steps):
        sim_t = t if time_rule == "accumulate" else 0.0 + n * dt
        try:
            engine.spring_pass(st, sim_t, cfg)
            counters += engine._cache_for(st).counters
            engine.mass_pass(st, env, cfg)
        except Exception as exc:  # NumericalAbort
            err = int(exc.mass_slot) + 1
            done = n + 1
            break
        t = t + dt
        done = n + 1
        if done in checkpoints:
            m, s = st.mass_slot_count, st.spring_slot_count
            out[f"{tag}pos_{done}"] = st._m_pos[:m].copy()
            out[f"{tag}vel_{done}"] = st._m_vel[:m].copy()
            out[f"{tag}acc_{done}"] = st._m_acc[:m].copy()
            out[f"{tag}s_alive_{done}"] = st._s_alive[:s].astype(np.uint8)
            out[f"{tag}counters_{done}"] = counters.copy()
    out[f"{tag}steps_done"] = np.int64(done)
    out[f"{tag}err_slot"] = np.int64(err)
    m, s = st.mass_slot_count, st.spring_slot_count
    out[f"{tag}final_pos"] = st._m_pos[:m].copy()
    out[f"{tag}final_vel"] = st._m_vel[:m].copy()
    out[f"{tag}final_acc"] = st._m_acc[:m].copy()
    out[f"{tag}final_fext"] = st._m_fext[:m].copy()
    out[f"{tag}final_s_alive"] = st._s_alive[:s].astype(np.uint8)
    out[f"{tag}final_s_degen"] = st._s_degen[:s].astype(np.uint8)
    out[f"{tag}final_counters"] = counters.copy()


def save(name, st_factory, env, dt, steps, checkpoints=(), time_rule="accumulate",
         check_slotted=True, meta=None):
    st = st_factory()
    case = store_case(st, env)
    case.update({"dt": np.float64(dt), "n_steps": np.int64(steps),
                 "time_rule": np.array(time_rule)})
    for k, v in (meta or {}).items():
        case[f"meta_{k}"] = np.asarray(v)
    run_reference(st, env, dt, steps, set(checkpoints), time_rule, case)
    if check_slotted:
        st2 = st_factory()
        chk = {}
        run_reference(st2, env, dt, steps, set(), time_rule, chk,
                      accumulation="slotted")
        assert np.array_equal(chk["final_pos"], case["final_pos"]), name
        assert np.array_equal(chk["final_vel"], case["final_vel"]), name
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **case)
    print(f"{name}: masses={len(case['m_mass'])} springs={len(case['s_m1'])}"
          f" steps={int(case['steps_done'])} err={int(case['err_slot'])} "
          f"counters={case['final_counters'].tolist()} -> "
          f"{os.path.getsize(path) / 1024:.0f} KiB")


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


def main():
    cube_mat = Material(elastic_modulus=1e6, density=1000.0)
    g = Vec3(0, 0, -9.81)

    # config A (pkg/scenarios/bouncing_cube.ini): controller time rule.
    env_a = Environment(gravity=g, contacts=[ground(2000.0, 1.0, 0.8)])
    save("cube10_drop",
         lambda: lattice(10, 0.1, cube_mat, corner=(0, 0, 0.3))[0],
         env_a, 1e-4, 1000, checkpoints=(100,), time_rule="index",
         meta={"n": 10, "spacing": 0.1, "E": 1e6, "rho": 1000.0,
               "corner": (0, 0, 0.3)})

    # config A in ground contact from step 0 (SURVEY 8(d) variant)
    save("cube10_contact",
         lambda: lattice(10, 0.1, cube_mat, corner=(0, 0, -0.002),
                         stretch=1.01)[0],
         env_a, 1e-4, 200, checkpoints=(100,), time_rule="index")

    # test_engine.py:400-421 case: 3^3, drag, contact
    env_c = Environment(gravity=g, drag_coeff=0.01,
                        contacts=[ground(500.0, 0.6, 0.5)])
    save("lat3_contact_drag",
         lambda: lattice(3, corner=(0, 0, 0.01), stretch=1.05)[0],
         env_c, 1e-4, 100, checkpoints=(1, 10, 100))

    # worm (pkg/scenarios/worm.ini / test_acceptance.py:297-326)
    def worm():
        st, body = lattice(0, 0.05, cube_mat, nxyz=(20, 6, 6))
        configure_worm(body, st)
        return st
    env_w = Environment(gravity=g, drag_coeff=0.01,
                        contacts=[ground(500.0, 1.0, 0.8)])
    save("worm", worm, env_w, 1e-4, 300, checkpoints=(100,),
         time_rule="index")

    # quiescent sine + explicit offsets, accumulate time rule
    def quiescent():
        st, body = lattice(4, stretch=1.02)
        for i, h in enumerate(body.spring_handles):
            st.set_spring_field(h, "actuation", ActuationParams(
                amplitude=0.3, frequency=50.0, offset=1e-3 * (i % 7),
                period=0.013, quiescent_before_offset=bool(i % 2)))
        return st
    save("actuated_quiescent", quiescent, Environment(gravity=g), 1e-4, 120,
         checkpoints=(7, 100))

    # yield breaking: nylon-like bars, stretched so some springs break
    nylon = Material(elastic_modulus=4.56e9, density=1150.0,
                     yield_stress=8e7)
    def yielding():
        st, body = lattice(4, spacing=0.01, mat=nylon, stretch=1.0)
        slots = body.mass_handles.slots
        x = st._m_pos[slots, 0]
        st._m_pos[slots, 0] = x * (1.0 + 0.05 * (x > 0.015))
        return st
    save("yield_break", yielding, Environment(gravity=Vec3(0, 0, 0)), 5e-9,
         60, checkpoints=(1, 2))

    # constraints, fixed masses, applied loads, balls, global constraint
    def constrained():
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
        return st
    env_k = Environment(gravity=g, drag_coeff=0.05, contacts=[
        ground(800.0, 0.7, 0.4),
        ContactPlane(normal=Vec3(1, 0, 0), offset=0.01, stiffness=300.0,
                     static_friction=0.2, kinetic_friction=0.1),
        ContactBall(center=Vec3(0.08, 0.08, 0.2), radius=0.12,
                    stiffness=400.0)])
    save("constraints_contacts", constrained, env_k, 1e-4, 150,
         checkpoints=(1, 50, 100))

    # topology edits: dead masses (lazy invalidation), deleted springs, LIFO
    # slot reuse, a degenerate (zero-length) spring
    def edited():
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
        st.create_spring(Spring(m1=hs[1], m2=a, rest_length=0.2,
                                stiffness=7.0))
        st.create_spring(Spring(m1=b, m2=hs[60], rest_length=0.2,
                                stiffness=7.0, diameter=1e-3,
                                yield_stress=1e3))
        return st
    save("topology_edits", edited, Environment(gravity=g), 1e-4, 120,
         checkpoints=(1, 100))

    # numerical abort (test_engine.py:160-168)
    def blowup():
        st = ObjectStore()
        a = st.create_mass(Mass(pos=Vec3(0, 0, 0), m=1.0))
        b = st.create_mass(Mass(pos=Vec3(1, 0, 0), m=1e-30))
        st.create_spring(Spring(m1=a, m2=b, rest_length=0.1, stiffness=1e30))
        return st
    save("nan_abort", blowup, Environment(gravity=Vec3(0, 0, 0)), 1.0, 50,
         check_slotted=False)


if __name__ == "__main__":
    main()
