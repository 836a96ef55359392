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


@pytest.mark.parametrize("cfg,dims", [(1, (384, 512, 6)), (3, (256, 256, 8))])
def test_track_properties_large(cfg, dims):
    """Size-independent properties at sizes the golden fixtures do not
    reach: the nodes are exactly the critical-face set, consecutive faces of
    a chain share a tet (an edge of the graph), the component count is
    verify()'s n_traj, and every crossing lies in the field's extent."""
    from paper_2510_25143_b200 import (build_critical_face_set, synth,
                                       to_fixed, verify)
    H, W, T = dims
    _, _, _, u, v = synth.generate(cfg, H, W, T)
    f = FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    g = tracking.extract_trajectories(f)
    cfs = build_critical_face_set(to_fixed(f))
    assert set(g.nodes) == set(cfs.members) and len(cfs.members) > 0
    assert sum(len(c) for c in g.components) == len(cfs.members)
    for k, chain in enumerate(g.components):
        for a, b in zip(chain, chain[1:]):
            assert tuple(sorted((a, b))) in g.edges
        if g.loops[k]:
            assert tuple(sorted((chain[0], chain[-1]))) in g.edges
    assert len(g.edges) == sum(len(c) - (0 if lp else 1)
                               for c, lp in zip(g.components, g.loops))
    rep = verify(f, f)
    assert rep.n_traj_orig == g.n_components and rep.isomorphic
    xyt = np.asarray(list(g.nodes.values()))
    assert (xyt[:, 0] >= 0).all() and (xyt[:, 0] <= W - 1).all()
    assert (xyt[:, 1] >= 0).all() and (xyt[:, 1] <= H - 1).all()
    assert (xyt[:, 2] >= 0).all() and (xyt[:, 2] <= T - 1).all()
