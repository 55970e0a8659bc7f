"""Reference-pinned device diagnostics and callable waveforms.

tests/golden/make_diag_golden.py ran the REFERENCE (softlat serial backend)
and recorded, at an instant of a run, the store state and the reference's
own ``engine.mechanical_energy`` / ``engine.spring_loads``
(/root/reference/pkg/src/softlat/engine.py:366-412).  The device
diagnostics (sl_energy, sl_spring_loads) are checked against those values
(fp64 mode: identical inputs; sums in another order, so 1e-12 relative).

``custom_wave``: springs with a CALLABLE waveform (store.py:40, 413-415),
whose factor the host evaluates every step (engine._fill_custom_factors,
engine.py:149-155) and ships to the device (sl_set_custom_factors).  The
same lattice built through this package's API and stepped 80 steps in fp64
must equal the reference's trajectory bit for bit.
"""
import math

import numpy as np
import pytest

from conftest import case_context, load_golden, rel_maxnorm
from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, StepConfig, Vec3, engine)
from paper_1911_10274_b200.actuation import ActuationParams
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice

pytestmark = pytest.mark.gpu

DIAG = ("diag_worm", "diag_quiescent", "diag_edits")


@pytest.mark.parametrize("precision", ["fp64", "fp32", "mixed"])
@pytest.mark.parametrize("name", DIAG)
def test_device_energy_matches_reference(name, precision):
    g = load_golden(name)
    ctx = case_context(g, precision)
    ke, spe, gpe = ctx.energy(float(g["sim_t"]), g["gravity"])
    ctx.close()
    # fp64 state: only the summation order differs; fp32 / mixed: the
    # state itself is rounded (compensated positions / fp32 rest lengths)
    tol = 1e-12 if precision == "fp64" else 1e-5
    for got, want in ((ke, g["e_kinetic"]), (spe, g["e_spring"]),
                      (gpe, g["e_gravity"])):
        assert abs(got - float(want)) <= tol * abs(float(want)), \
            (name, got, float(want))


@pytest.mark.parametrize("name", DIAG)
def test_device_spring_loads_match_reference(name):
    g = load_golden(name)
    ctx = case_context(g, "fp64")
    n = len(g["s_m1"])
    lengths, fmag = ctx.spring_loads(float(g["sim_t"]), n)
    ctx.close()
    slots = g["loads_slots"]
    alive = np.flatnonzero(~np.isnan(lengths))
    assert np.array_equal(alive, slots)  # dead slots excluded, as the ref
    assert np.allclose(lengths[slots], g["loads_len"], rtol=1e-14, atol=0)
    # |k (|d| - f L0)| cancels: compare on the scale of the loads
    scale = float(np.abs(g["loads_fmag"]).max())
    assert np.abs(fmag[slots] - g["loads_fmag"]).max() <= 1e-9 * scale
    # the stress the host forms from them (engine.spring_loads)
    area = 0.25 * np.pi * g["s_diam"][slots] ** 2
    stress = fmag[slots] / area
    ok = np.isfinite(g["loads_stress"])
    assert np.allclose(stress[ok], g["loads_stress"][ok], rtol=1e-9,
                       atol=1e-9 * float(np.abs(g["loads_stress"][ok]).max()))


def custom_waveform(t: float) -> float:
    """Same function as tests/golden/make_diag_golden.py custom_waveform."""
    return 1.0 + 0.15 * math.sin(37.0 * t) * math.cos(11.0 * t) + 0.4 * t


def _custom_store():
    st = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0.05), 5, 5, 5, 0.05,
                                     Material(1e5, 1000.0)), st)
    st._m_pos[body.mass_handles.slots] *= 1.01
    for i, h in enumerate(body.spring_handles):
        if i % 3 == 0:
            st.set_spring_field(h, "actuation", ActuationParams(
                amplitude=0.0, frequency=0.0, offset=2e-3 * (i % 5),
                period=0.02, waveform=custom_waveform))
    env = Environment(gravity=Vec3(0, 0, -9.81), contacts=[ContactPlane(
        normal=Vec3(0, 0, 1), offset=0.0, stiffness=800.0,
        static_friction=0.9, kinetic_friction=0.7)])
    return st, env


def test_custom_waveform_store_matches_golden_inputs():
    g = load_golden("custom_wave")
    st, _ = _custom_store()
    m, s = st.mass_slot_count, st.spring_slot_count
    assert st._m_pos[:m].tobytes() == g["m_pos"].tobytes()
    assert np.array_equal(st._s_act_mode[:s], g["s_mode"])
    assert (g["s_mode"] == 3).sum() > 0


@pytest.mark.parametrize("split", [(80,), (40, 40), (13, 27, 40)])
def test_custom_waveform_fp64_bit_exact(split):
    """Callable factors pushed from the host every step (1-step launches),
    run in one or several engine calls: the reference's trajectory."""
    g = load_golden("custom_wave")
    st, env = _custom_store()
    cfg = StepConfig(dt=float(g["dt"]))
    done = 0
    for n in split:
        engine.run_steps(st, env, cfg, n, time_rule="index", step0=done)
        done += n
        if done == 40:
            m = st.mass_slot_count
            assert st._m_pos[:m].tobytes() == g["pos_40"].tobytes()
    m = st.mass_slot_count
    assert st._m_pos[:m].tobytes() == g["final_pos"].tobytes()
    assert st._m_vel[:m].tobytes() == g["final_vel"].tobytes()


@pytest.mark.parametrize("precision", ["fp32", "mixed"])
def test_custom_waveform_reduced_precision(precision):
    g = load_golden("custom_wave")
    st, env = _custom_store()
    engine.run_steps(st, env, StepConfig(dt=float(g["dt"]),
                                         precision=precision), 80,
                     time_rule="index")
    m = st.mass_slot_count
    assert rel_maxnorm(st._m_pos[:m], g["final_pos"]) < 1e-4
    assert rel_maxnorm(st._m_vel[:m], g["final_vel"]) < 1e-4


def test_custom_waveform_controller_matches_golden():
    """The SimController path (control.py: one-step batches while custom
    waveforms exist) reproduces the same 80 steps."""
    from paper_1911_10274_b200.control import SimController
    g = load_golden("custom_wave")
    st, env = _custom_store()
    ctl = SimController(st, env, StepConfig(dt=float(g["dt"])))
    ctl.start(80 * float(g["dt"]))
    rep = ctl.wait_for_event(timeout=60)
    assert rep.step_count == 80
    m = st.mass_slot_count
    assert st._m_pos[:m].tobytes() == g["final_pos"].tobytes()
    ctl.stop()
