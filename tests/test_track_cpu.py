"""Trajectory extraction host logic (linking, chain order, exact crossing
points, CSV) against the reference's own outputs (tests/golden/track_*.npz,
oracle/gen_track_golden.py).  The positive faces come from the source
fixture's golden critical-face set, so no GPU is needed."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2510_25143_b200 import tracking
from paper_2510_25143_b200.field import round_half_away
from paper_2510_25143_b200.predicates import mask_to_faces

GOLD = Path(__file__).parent / "golden"
CASES = sorted(GOLD.glob("track_*.npz"))


def golden_chains(z):
    comp, faces = z["comp"], z["faces"]
    chains = [[] for _ in range(len(z["loop"]))]
    for k, f in zip(comp.tolist(), faces.tolist()):
        chains[k].append(tuple(f))
    return chains


def host_graph(z):
    src = np.load(GOLD / str(z["source"]))
    H, W, T = int(src["H"]), int(src["W"]), int(src["T"])
    n = H * W * T
    mask = np.zeros(n, np.uint16)
    mask[src["mask_anchor"]] = src["mask_bits"]
    sl, sb = mask_to_faces(mask, H, W, T)
    faces = sl | sb
    s = float(src["scale"])
    uf = round_half_away(src["u"].astype(np.float64) * s)
    vf = round_half_away(src["v"].astype(np.float64) * s)
    fixed = {w: (int(uf[w]), int(vf[w])) for fc in faces for w in fc}
    return tracking.trajectories_from_faces(
        faces, fixed, H, W, T, float(src["dx"]), float(src["dy"]),
        float(src["dt"]))


def check_graph(g, z):
    ref = golden_chains(z)
    assert g.n_components == len(ref)
    assert g.loops == z["loop"].tolist()
    # chains exactly, closed loops' direction included
    assert g.components == ref
    # exact crossing points (bitwise float64)
    for f, xyt in zip(z["faces"].tolist(), z["xyt"]):
        assert np.array_equal(np.asarray(g.nodes[tuple(f)]), xyt), f


@pytest.mark.parametrize("path", CASES, ids=lambda p: p.stem)
def test_track_host_matches_reference(path, tmp_path):
    z = np.load(path)
    g = host_graph(z)
    check_graph(g, z)
    out = tmp_path / "t.csv"
    tracking.write_trajectory_csv(g, out)
    assert out.read_text() == str(z["csv"])


def test_track_fixtures_present():
    assert len(CASES) >= 10
    assert any(np.load(p)["loop"].any() for p in CASES)


def test_topology_error_on_dangling_face():
    # a lone slab face: its tets each see one crossed face
    H = W = T = 3
    f = (0, 1, 1 + H * W)
    with pytest.raises(tracking.TopologyError):
        tracking.ordered_components({f}, H, W, T)


def test_loop_orientation_is_deterministic():
    z = np.load(next(p for p in CASES if np.load(p)["loop"].any()))
    a, b = host_graph(z), host_graph(z)
    assert a.components == b.components
