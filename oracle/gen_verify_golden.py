"""Golden VerifyReports from the reference itself (tracking.py:170-195).

Runs the reference package (importable in the build container, not on the
GPU box) on golden fields: the original vs its reference reconstruction
(trajectories preserved), and vs a seeded perturbation of it (faces flip).
Writes tests/golden/verify.json.  The test rebuilds the same inputs.

    PYTHONPATH=/root/reference/pkg/src python oracle/gen_verify_golden.py
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
from vfcp.field import FieldSeries  # noqa: E402  (the reference)
from vfcp.tracking import verify  # noqa: E402

NAMES = ["vortex_small", "cfg1_eps0.01", "moving_vortex_mop", "int3",
         "vortex_pair_mop"]


def inputs(g, perturb):
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


def main():
    out = {}
    for name in NAMES:
        g = dict(np.load(ROOT / "tests" / "golden" / f"field_{name}.npz"))
        for perturb in (False, True):
            H, W, T, S, ru, rv = inputs(g, perturb)
            fo = FieldSeries(H, W, T, float(g["dx"]), float(g["dy"]),
                             float(g["dt"]), g["u"], g["v"])
            fr = FieldSeries(H, W, T, float(g["dx"]), float(g["dy"]),
                             float(g["dt"]), ru, rv)
            key = f"{name}/{'perturbed' if perturb else 'recon'}"
            try:
                r = verify(fo, fr, archive_size=len(bytes(g["archive"])), scale=S)
            except Exception as e:   # the reference's own error, e.g. TopologyError
                out[key] = {"error": type(e).__name__}
                print(name, perturb, out[key])
                continue
            out[key] = {
                "cr": r.cr, "psnr": r.psnr, "max_abs_err": r.max_abs_err,
                "fc_t": r.fc_t, "fc_s": r.fc_s, "n_traj_orig": r.n_traj_orig,
                "n_traj_recon": r.n_traj_recon, "isomorphic": r.isomorphic}
            print(name, perturb, out[key])
    (ROOT / "tests" / "golden" / "verify.json").write_text(
        json.dumps(out, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()
