"""extract_trajectories on the device path (face mask from the analysis
kernel, fixed-point gather on the device) against the reference's own
trajectories (tests/golden/track_*.npz, oracle/gen_track_golden.py)."""

from pathlib import Path

import numpy as np
import pytest

from paper_2510_25143_b200 import FieldSeries, tracking
from test_track_cpu import CASES, check_graph

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


@pytest.mark.parametrize("path", CASES, ids=lambda p: p.stem)
def test_track_device_matches_reference(path, tmp_path):
    z = np.load(path)
    src = np.load(GOLD / str(z["source"]))
    f = FieldSeries(int(src["H"]), int(src["W"]), int(src["T"]),
                    float(src["dx"]), float(src["dy"]), float(src["dt"]),
                    src["u"], src["v"])
    g = tracking.extract_trajectories(f)
    check_graph(g, z)
    out = tmp_path / "t.csv"
    tracking.write_trajectory_csv(g, out)
    assert out.read_text() == str(z["csv"])
