"""Golden ResidualStats from the reference itself (tracking.py:228-268).

Runs the reference's residual_stats (importable in the build container, not
on the GPU box) on seeded symbol streams -- geometric residuals around the
radius with escapes, long center runs, an all-center and an empty stream --
and writes tests/golden/residual_stats.npz (inputs and outputs).

    python oracle/gen_residual_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
from vfcp.tracking import residual_stats  # noqa: E402  (the reference)


def streams():
    rng = np.random.default_rng(11)
    out = {}
    for k, (radius, n, p_esc) in enumerate([(16, 3000, 0.02), (4, 500, 0.2),
                                            (32768, 20000, 0.001)]):
        mag = rng.geometric(0.6, n) - 1
        sgn = rng.choice([-1, 1], n)
        s = np.clip(radius + mag * sgn, 1, 2 * radius - 1)
        s[rng.random(n) < p_esc] = 0
        out[f"s{k}"] = (s.astype(np.int64), radius)
    out["center"] = (np.full(64, 8, np.int64), 8)
    out["empty"] = (np.zeros(0, np.int64), 8)
    out["escapes"] = (np.zeros(10, np.int64), 8)
    return out


def main():
    arrs = {}
    for name, (s, radius) in streams().items():
        r = residual_stats(s, radius)
        arrs[f"{name}_sym"] = s
        arrs[f"{name}_radius"] = np.int64(radius)
        arrs[f"{name}_pmf"] = r.folded_pmf
        arrs[f"{name}_ccdf"] = r.tail_ccdf
        arrs[f"{name}_ov"] = np.float64(r.overflow_rate)
        arrs[f"{name}_runs"] = r.run_lengths
        arrs[f"{name}_run_ccdf"] = r.run_ccdf
        arrs[f"{name}_run_mean"] = np.float64(r.run_mean)
        arrs[f"{name}_pct"] = np.array([r.run_percentiles[q] for q in (75, 80, 85, 90)])
    np.savez_compressed(ROOT / "tests" / "golden" / "residual_stats.npz", **arrs)


if __name__ == "__main__":
    main()
