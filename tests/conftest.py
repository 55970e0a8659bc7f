"""Shared pytest configuration.

Markers: ``gpu`` tests need a B200 (run on the GPU box via gpurun); all other
tests run on the CPU-only build container.
"""
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
for p in (ROOT, os.path.join(ROOT, "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running test")


GOLDEN_CASES = ("cube10_drop", "cube10_contact", "lat3_contact_drag", "worm",
                "actuated_quiescent", "yield_break", "constraints_contacts",
                "topology_edits", "nan_abort")


def load_golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"{name}.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def golden():
    return load_golden


def have_gpu() -> bool:
    try:
        from paper_1911_10274_b200 import _native
        return _native.device_count() > 0
    except Exception:
        return False


def case_context(case: dict, precision: str = "fp64", device: int = 0):
    """Upload a golden-format case through the C ABI (ctypes Context)."""
    from paper_1911_10274_b200 import _native
    ctx = _native.Context(device, precision)
    ctx.upload_masses(case["m_pos"], case["m_vel"], case["m_acc"],
                      case["m_fext"], case["m_load"], case["m_mass"],
                      case["m_fixed"], case["m_alive"], case["m_gen"])
    ctx.upload_springs(case["s_m1"], case["s_m2"], case["s_m1gen"],
                       case["s_m2gen"], case["s_rest"], case["s_k"],
                       case["s_diam"], case["s_yield"], case["s_mode"],
                       case["s_amp"], case["s_freq"], case["s_off"],
                       case["s_per"], case["s_alive"], case["s_degen"])
    ctx.set_local_constraints(case["lc_off"], case["lc_kind"],
                              case["lc_vec"])
    ctx.set_environment(case["gravity"], float(np.asarray(case["drag"])),
                        case["planes"], case["balls"], case["gc_kind"],
                        case["gc_vec"], 1e-6)
    return ctx


def case_times(case: dict) -> np.ndarray:
    from paper_1911_10274_b200.engine import step_times
    return step_times(int(case["n_steps"]), float(case["dt"]), 0.0,
                      str(case["time_rule"]))


def rel_maxnorm(got: np.ndarray, want: np.ndarray) -> float:
    """max|got-want| / max|want| (SURVEY.md 7 hard part 3: elementwise
    relative error is ill-posed where the reference holds exact zeros)."""
    scale = float(np.max(np.abs(want))) or 1.0
    return float(np.max(np.abs(got - want))) / scale
