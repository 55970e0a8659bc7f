"""Acceptance run of the reference (pkg/tests/test_acceptance.py:297-326):
a worm-actuated 20x6x6 body crawls for three actuation periods (30,000
steps) through SimController; the reference records a centre-of-mass
displacement of +0.4186 m (pkg/test_output.txt:36) and |dx| < 1e-6 for the
unactuated control."""
import pytest

from paper_1911_10274_b200 import (ContactPlane, Environment, Material,
                                   ObjectStore, StepConfig, Vec3)
from paper_1911_10274_b200.actuation import configure_worm
from paper_1911_10274_b200.builder import LatticeSpec, build_lattice
from paper_1911_10274_b200.control import SimController

pytestmark = pytest.mark.gpu

RECORDED_DX = 0.4186  # reference run, pkg/test_output.txt:36


def _worm_run(amplitude, precision):
    store = ObjectStore()
    body = build_lattice(LatticeSpec(Vec3(0, 0, 0), 20, 6, 6, 0.05,
                                     Material(1e6, 1000.0)), store)
    configure_worm(body, store, amplitude=amplitude)
    env = Environment(gravity=Vec3(0, 0, -9.81), drag_coeff=0.01,
                      contacts=[ContactPlane(
                          normal=Vec3(0, 0, 1), offset=0.0, stiffness=500.0,
                          static_friction=1.0, kinetic_friction=0.8)])
    ctl = SimController(store, env, StepConfig(dt=1e-4, precision=precision))
    com0 = body.center_of_mass(store).x
    ctl.start(3.0)
    rep = ctl.wait_for_event()
    assert rep.reason == "breakpoint", rep
    assert rep.step_count == 30000
    dx = body.center_of_mass(store).x - com0
    ctl.stop()
    return dx


@pytest.mark.parametrize("precision", ["fp64", "mixed", "fp32"])
def test_worm_locomotion(precision):
    dx = _worm_run(0.2, precision)
    assert dx > 0
    assert abs(dx - RECORDED_DX) < 5e-3 * RECORDED_DX, dx
    assert abs(_worm_run(0.0, precision)) < 1e-6
