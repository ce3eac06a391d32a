"""goomjac v1 I/O (lyapunov.py:433-476) — host code, no GPU: a file the
reference wrote loads to the same chain, round trips are exact, malformed files raise."""

import os

import numpy as np
import pytest

from goom_testlib import GOLDEN, load_golden


@pytest.fixture(scope="module")
def lyap():
    from paper_2510_03426_b200 import lyapunov

    return lyapunov


def test_reads_reference_file_and_round_trips(lyap, tmp_path):
    z = load_golden("goomjac_ref")
    ch = lyap.load_jacobian_chain(os.path.join(GOLDEN, "chain_ref.goomjac"))
    np.testing.assert_array_equal(ch.mats, z["mats"])
    assert ch.dt == float(z["dt"])
    p = tmp_path / "c.goomjac"
    lyap.save_jacobian_chain(ch, p)
    assert p.read_text() == open(os.path.join(GOLDEN, "chain_ref.goomjac")).read()
    again = lyap.load_jacobian_chain(p)
    np.testing.assert_array_equal(again.mats, ch.mats)


@pytest.mark.parametrize("text", [
    "",
    "goomjac v2 d=2 T=1 dt=1.0\n1 0\n0 1\n",
    "goomjac v1 d=2 T=1 dt=1.0\n1 0\n0 1\nextra\n",
    "goomjac v1 d=2 T=1 dt=1.0\n1 0\n0\n",
    "goomjac v1 d=2 T=1 dt=0\n1 0\n0 1\n",
    "goomjac v1 d=2 T=1\n1 0\n0 1\n",
    "goomjac v1 d=2 T=1 dt=1.0\n1 nan\n0 1\n",
])
def test_malformed_files_raise(lyap, tmp_path, text):
    p = tmp_path / "bad.goomjac"
    p.write_text(text)
    with pytest.raises(ValueError):
        lyap.load_jacobian_chain(p)
