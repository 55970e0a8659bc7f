"""Snapshot / energy-log files (io.py of the reference) on CPU: the native
formatter is byte-identical to the reference's own format_snapshot on the
committed golden rows (tests/golden/make_io_golden.py ran the reference),
the reader round-trips bit-exactly and raises the reference's errors."""
import os

import numpy as np
import pytest

from paper_1911_10274_b200 import ObjectStore, Vec3, Mass
from paper_1911_10274_b200 import io as sio
from paper_1911_10274_b200.errors import ScenarioError

GOLD = os.path.join(os.path.dirname(__file__), "golden", "snapshot_io.npz")


@pytest.fixture(scope="module")
def gold():
    with np.load(GOLD) as z:
        return {k: z[k] for k in z.files}


def test_format_matches_reference_bytes(gold):
    out = bytes(sio.format_snapshot_bytes(gold["ids"], gold["pos"],
                                          gold["vel"]))
    assert out == gold["text"].tobytes()
    assert sio.format_snapshot(np.zeros(0, np.int64), np.zeros((0, 3)),
                               np.zeros((0, 3))) == gold["empty"].tobytes(
                                   ).decode()


def _py_format(ids, pos, vel):
    """io.py:19-27 restated (the checker for the threaded chunking)."""
    lines = [sio.SNAPSHOT_HEADER]
    for i in range(len(ids)):
        x, y, z = pos[i]
        vx, vy, vz = vel[i]
        lines.append(f"{int(ids[i])},{x:.17g},{y:.17g},{z:.17g},"
                     f"{vx:.17g},{vy:.17g},{vz:.17g}")
    return "\n".join(lines) + "\n"


@pytest.mark.parametrize("n", [1, 4095, 4097, 40000])
def test_threaded_chunks_match_python_loop(n):
    rng = np.random.default_rng(n)
    ids = rng.integers(0, 10 ** 9, n)
    pos = rng.normal(0, 3, (n, 3))
    vel = rng.normal(0, 1e-3, (n, 3))
    assert sio.format_snapshot(ids, pos, vel) == _py_format(ids, pos, vel)


def test_write_read_roundtrip_bit_exact(tmp_path, gold):
    p = tmp_path / "snap.csv"
    sio.write_snapshot(p, gold["ids"], gold["pos"], gold["vel"])
    ids, pos, vel = sio.read_snapshot(p)
    assert np.array_equal(ids, gold["ids"])
    for got, want in ((pos, gold["pos"]), (vel, gold["vel"])):
        fin = np.isfinite(want)
        assert got[fin].tobytes() == want[fin].tobytes()
        assert np.array_equal(np.isnan(got), np.isnan(want))
        assert np.array_equal(got[np.isinf(want)], want[np.isinf(want)])
    p2 = tmp_path / "snap.npz"
    sio.write_snapshot_npz(p2, gold["ids"], gold["pos"], gold["vel"])
    b = sio.read_snapshot_npz(p2)
    assert all(x.tobytes() == y.tobytes() for x, y in
               zip(b, (gold["ids"], gold["pos"], gold["vel"])))


def test_reader_errors_follow_the_reference(tmp_path):
    def write(text):
        p = tmp_path / "s.csv"
        p.write_text(text)
        return p
    h = sio.SNAPSHOT_HEADER + "\n"
    with pytest.raises(ScenarioError, match="bad header"):
        sio.read_snapshot(write("id,x,y\n1,2,3\n"))
    with pytest.raises(ScenarioError, match="bad header"):
        sio.read_snapshot(write(""))
    with pytest.raises(ScenarioError, match=":3: expected 7 columns"):
        sio.read_snapshot(write(h + "1,0,0,0,0,0,0\n2,0,0,0,0,0\n"))
    with pytest.raises(ScenarioError, match=":3: expected 7 columns"):
        sio.read_snapshot(write(h + "1,0,0,0,0,0,0\n\n2,0,0,0,0,0,0\n"))
    with pytest.raises(ValueError):  # float("0#") fails in the reference
        sio.read_snapshot(write(h + "1,0,0,0,0,0,0#\n"))
    ids, pos, vel = sio.read_snapshot(write(h))
    assert ids.shape == (0,) and pos.shape == (0, 3)
    ids, pos, vel = sio.read_snapshot(write(h + " 7, 1e-3,inf,-0,nan,2,3 \r\n"))
    assert ids.tolist() == [7] and pos[0, 0] == 1e-3 and np.isinf(pos[0, 1])
    assert np.signbit(pos[0, 2]) and np.isnan(vel[0, 0])


def test_apply_snapshot_checks_alive_slots():
    st = ObjectStore()
    hs = [st.create_mass(Mass(pos=Vec3(i, 0, 0), m=1.0)) for i in range(3)]
    st.delete_mass(hs[1])
    with pytest.raises(ScenarioError):
        sio.apply_snapshot(st, np.array([1]), np.zeros((1, 3)),
                           np.zeros((1, 3)))
    sio.apply_snapshot(st, np.array([2]), np.ones((1, 3)), np.ones((1, 3)))
    assert st._m_pos[2].tolist() == [1.0, 1.0, 1.0]
