"""Host builder on CPU: the library's threaded
lattice generator (sl_build_lattice) produces a store bit-identical to the
numpy restatement of builder.py:112-186 (itself pinned to the reference's
golden inputs by tests/test_host_parity.py), and bulk creates keep the
slot semantics when freed slots are reused."""
import numpy as np
import pytest

from paper_1911_10274_b200 import Mass, Material, ObjectStore, Vec3
from paper_1911_10274_b200.builder import (LatticeSpec, build_lattice,
                                           build_lattice_numpy,
                                           lattice_spring_count)

M_COLS = ("_m_pos", "_m_vel", "_m_acc", "_m_fext", "_m_load", "_m_mass",
          "_m_fixed", "_m_alive", "_m_gen")
S_COLS = ("_s_m1", "_s_m2", "_s_m1gen", "_s_m2gen", "_s_rest", "_s_k",
          "_s_diam", "_s_yield", "_s_act_mode", "_s_alive", "_s_booked",
          "_s_degen", "_s_gen")


def same_store(a, b):
    assert a.mass_slot_count == b.mass_slot_count
    assert a.spring_slot_count == b.spring_slot_count
    for k in M_COLS:
        assert getattr(a, k)[:a.mass_slot_count].tobytes() == \
            getattr(b, k)[:b.mass_slot_count].tobytes(), k
    for k in S_COLS:
        assert getattr(a, k)[:a.spring_slot_count].tobytes() == \
            getattr(b, k)[:b.spring_slot_count].tobytes(), k


@pytest.mark.parametrize("dims,corner,spacing,diam", [
    ((1, 1, 1), (0, 0, 0), 0.1, 1e-3),
    ((5, 1, 1), (0, 0, 0), 0.1, 1e-3),
    ((2, 2, 2), (-1.5, 0.25, 3e-3), 0.05, 1e-3),
    ((7, 3, 11), (0.1, -0.3, 0.01), 0.037, 2.5e-3),
    ((1, 9, 4), (1e3, 0, -2), 1.1, 0.0),
    ((23, 17, 29), (0, 0, 0), 0.05, 1e-3)])
def test_native_lattice_identical_to_numpy(dims, corner, spacing, diam):
    mat = Material(elastic_modulus=1e6, density=1000.0, yield_stress=3e8)
    spec = LatticeSpec(Vec3(*corner), *dims, spacing, mat, diam)
    a, b = ObjectStore(), ObjectStore()
    ba = build_lattice(spec, a)
    bb = build_lattice_numpy(spec, b)
    same_store(a, b)
    assert a.spring_slot_count == lattice_spring_count(*dims)
    assert np.array_equal(ba.grid_indices, bb.grid_indices)
    assert ba.initial_positions.tobytes() == bb.initial_positions.tobytes()


def test_bulk_create_reuses_freed_slots_lifo():
    mat = Material(elastic_modulus=1e5, density=1000.0)
    spec = LatticeSpec(Vec3(0, 0, 0), 3, 3, 3, 0.05, mat)
    a, b = ObjectStore(), ObjectStore()
    for st in (a, b):
        hs = [st.create_mass(Mass(pos=Vec3(i, 0, 5), m=1.0)) for i in range(6)]
        for h in hs[1:4]:
            st.delete_mass(h)
    build_lattice(spec, a)
    build_lattice_numpy(spec, b)
    same_store(a, b)
    # the three freed slots were reused first (LIFO), then fresh ones
    assert a.mass_slot_count == 6 + 27 - 3
