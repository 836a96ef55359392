"""tracking.verify on the device vs the reference's own VerifyReports
(tests/golden/verify.json, made by oracle/gen_verify_golden.py from the
reference): reconstructions that keep every trajectory, and seeded
perturbations that flip faces and split trajectories."""
import json
from pathlib import Path

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "verify.json").read_text())


def _inputs(g, perturb):
    # the same inputs as oracle/gen_verify_golden.py
    H, W, T = int(g["H"]), int(g["W"]), int(g["T"])
    S = float(g["scale"])
    ru = g["recon"][0].reshape(-1).astype(np.int64) * (1.0 / S)
    rv = g["recon"][1].reshape(-1).astype(np.int64) * (1.0 / S)
    if perturb:
        rng = np.random.default_rng(12345)
        amp = 3.0 * float(g["eps_abs"])
        ru = ru + amp * rng.standard_normal(ru.size)
        rv = rv + amp * rng.standard_normal(rv.size)
    return H, W, T, S, ru, rv


@pytest.mark.parametrize("key", sorted(GOLD))
def test_verify_matches_reference(key):
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200 import tracking
    name, kind = key.split("/")
    g = load_golden(name)
    H, W, T, S, ru, rv = _inputs(g, kind == "perturbed")
    fo = vg.FieldSeries(H, W, T, float(g["dx"]), float(g["dy"]), float(g["dt"]),
                        g["u"], g["v"])
    fr = vg.FieldSeries(H, W, T, float(g["dx"]), float(g["dy"]), float(g["dt"]),
                        ru, rv)
    ref = GOLD[key]
    if "error" in ref:
        with pytest.raises(tracking.TopologyError):
            tracking.verify(fo, fr, archive_size=len(bytes(g["archive"])), scale=S)
        return
    r = tracking.verify(fo, fr, archive_size=len(bytes(g["archive"])), scale=S)
    for k in ("fc_t", "fc_s", "n_traj_orig", "n_traj_recon", "isomorphic"):
        assert getattr(r, k) == ref[k], k
    assert r.cr == ref["cr"] and r.max_abs_err == ref["max_abs_err"]
    # the device mean sums in another order than numpy's pairwise sum
    assert r.psnr == pytest.approx(ref["psnr"], rel=1e-10, abs=0.0)
    assert r.ok == (kind == "recon")
