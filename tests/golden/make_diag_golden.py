"""Reference-produced goldens for the device diagnostics and for callable
waveforms.

Run in the build container only (needs /root/reference and numba):

    python tests/golden/make_diag_golden.py

* ``diag_*.npz``: a case stepped by the reference's serial backend to some
  instant, then the store at that instant (``store_case``) together with
  the reference's own ``engine.mechanical_energy(store, env, sim_t)`` and
  ``engine.spring_loads(store, sim_t)`` (engine.py:366-412) there.
* ``custom_wave.npz``: a lattice whose springs carry a CALLABLE waveform
  (store.py:40, 413-415; filled on the host every step by
  engine._fill_custom_factors, engine.py:149-155), stepped 80 steps.  The
  waveform is ``custom_waveform`` below; tests/test_gpu_goldens_diag.py
  defines the same function.

Nothing on the GPU box reads /root/reference.
"""
from __future__ import annotations

import math
import os

import numpy as np

import make_golden as mg  # noqa: E402  (sets up the reference import)
from softlat import Environment, Vec3, engine  # noqa: E402
from softlat.actuation import ActuationParams  # noqa: E402


def custom_waveform(t: float) -> float:
    """Rest-length factor of the callable-waveform golden (local time t)."""
    return 1.0 + 0.15 * math.sin(37.0 * t) * math.cos(11.0 * t) + 0.4 * t


def diag(name, st_factory, env, dt, steps, time_rule):
    st = st_factory()
    out = {}
    mg.run_reference(st, env, dt, steps, set(), time_rule, out)
    assert int(out["err_slot"]) == 0
    sim_t = (steps * dt) if time_rule == "index" else float(
        sum([dt] * steps))
    if time_rule != "index":  # accumulated exactly as run_reference
        t = 0.0
        for _ in range(steps):
            t = t + dt
        sim_t = t
    case = mg.store_case(st, env)
    e = engine.mechanical_energy(st, env, sim_t)
    loads = engine.spring_loads(st, sim_t)
    case.update({"sim_t": np.float64(sim_t),
                 "e_kinetic": np.float64(e.kinetic),
                 "e_spring": np.float64(e.spring_potential),
                 "e_gravity": np.float64(e.gravity_potential),
                 "loads_slots": np.asarray(loads.slots, np.int64),
                 "loads_len": loads.lengths, "loads_fmag": loads.force_magnitudes,
                 "loads_stress": loads.stresses})
    path = os.path.join(mg.HERE, f"{name}.npz")
    np.savez_compressed(path, **case)
    print(f"{name}: t={sim_t:g} E=({e.kinetic:.6g}, {e.spring_potential:.6g},"
          f" {e.gravity_potential:.6g}) springs={len(loads.slots)}")


def main():
    g = Vec3(0, 0, -9.81)
    cube_mat = mg.Material(elastic_modulus=1e6, density=1000.0)

    def worm():
        st, body = mg.lattice(0, 0.05, cube_mat, nxyz=(20, 6, 6))
        mg.configure_worm(body, st)
        return st
    env_w = Environment(gravity=g, drag_coeff=0.01,
                        contacts=[mg.ground(500.0, 1.0, 0.8)])
    diag("diag_worm", worm, env_w, 1e-4, 150, "index")

    def quiescent():
        st, body = mg.lattice(4, stretch=1.02)
        for i, h in enumerate(body.spring_handles):
            st.set_spring_field(h, "actuation", ActuationParams(
                amplitude=0.3, frequency=50.0, offset=1e-3 * (i % 7),
                period=0.013, quiescent_before_offset=bool(i % 2)))
        return st
    diag("diag_quiescent", quiescent, Environment(gravity=g), 1e-4, 60,
         "accumulate")

    def edited():
        st, body = mg.lattice(4, stretch=1.04)
        hs = list(body.mass_handles)
        sh = list(body.spring_handles)
        st.delete_mass(hs[6])
        st.delete_mass(hs[21])
        for i in (3, 40, 41, 100):
            st.delete_spring(sh[i])
        return st
    diag("diag_edits", edited, Environment(gravity=g), 1e-4, 50, "index")

    # callable waveforms (ACT_CUSTOM): every third spring
    def custom():
        st, body = mg.lattice(5, stretch=1.01, corner=(0, 0, 0.05))
        for i, h in enumerate(body.spring_handles):
            if i % 3 == 0:
                st.set_spring_field(h, "actuation", ActuationParams(
                    amplitude=0.0, frequency=0.0, offset=2e-3 * (i % 5),
                    period=0.02, waveform=custom_waveform))
        return st
    env_c = Environment(gravity=g, contacts=[mg.ground(800.0, 0.9, 0.7)])
    mg.save("custom_wave", custom, env_c, 1e-4, 80, checkpoints=(40,),
            time_rule="index", check_slotted=True)


if __name__ == "__main__":
    main()
