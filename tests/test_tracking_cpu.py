"""Trajectory linking (tracking.trajectory_graph) on the CPU: crossed faces
from the C oracle's exact / SoS predicate, trajectory counts against the
reference's own VerifyReports (tests/golden/verify.json)."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "verify.json").read_text())


def _fixed(x, S):
    y = np.asarray(x, np.float64) * S
    return (np.sign(y) * np.floor(np.abs(y) + 0.5)).astype(np.int64)


def _inputs(g, perturb):
    # as oracle/gen_verify_golden.py
    S = float(g["scale"])
    ru = g["recon"][0].reshape(-1).astype(np.int64) * (1.0 / S)
    rv = g["recon"][1].reshape(-1).astype(np.int64) * (1.0 / S)
    if perturb:
        rng = np.random.default_rng(12345)
        amp = 3.0 * float(g["eps_abs"])
        ru = ru + amp * rng.standard_normal(ru.size)
        rv = rv + amp * rng.standard_normal(rv.size)
    return S, ru, rv


@pytest.mark.parametrize("key", sorted(GOLD))
def test_trajectory_counts_match_reference(key, oracle_mod):
    from paper_2510_25143_b200 import tracking
    name, kind = key.split("/")
    ref = GOLD[key]
    if "error" in ref:
        pytest.skip("reference raised")
    g = load_golden(name)
    H, W, T = int(g["H"]), int(g["W"]), int(g["T"])
    S, ru, rv = _inputs(g, kind == "perturbed")
    for u, v, want in ((g["u"], g["v"], ref["n_traj_orig"]),
                       (ru, rv, ref["n_traj_recon"])):
        mask, _ = oracle_mod.analyze(H, W, T, _fixed(u, S), _fixed(v, S), 0,
                                     want_mask=True, want_xi=False)
        sl, sb = oracle_mod.mask_to_faces(mask, H, W, T)
        _, n = tracking.trajectory_graph(sl | sb, H, W, T)
        assert n == want


def test_topology_error_on_a_dangling_face():
    from paper_2510_25143_b200 import tracking
    # one crossed face alone: its tets have a single crossed face
    with pytest.raises(tracking.TopologyError):
        tracking.trajectory_graph({(0, 1, 6)}, 5, 5, 3)
