"""Golden CompressStats from the reference itself (codec.py:388-397).

Runs the reference's compress with Config(stats=True) (importable in the
build container, not on the GPU box) on a selection of the golden field
fixtures and writes tests/golden/compress_stats.npz: per field the stats'
symbols, signed_indices, overflow_count, lossless_vertices, modes and
critical_faces.  Test infrastructure only.

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/vfcp_numba python oracle/gen_stats_golden.py
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
import vfcp  # noqa: E402  (the reference)

GOLDEN = ROOT / "tests" / "golden"
FIELDS = ("cfg1_eps0.01", "cfg3_eps0.001", "escapes_radius4",
          "escapes_radius2_sl", "int60", "int3", "recompress_f64", "vortex_pair_mop",
          "random_fourier_lorenzo", "zero_eps")


def main():
    out = {}
    for name in FIELDS:
        z = np.load(GOLDEN / f"field_{name}.npz")
        f = vfcp.FieldSeries(int(z["H"]), int(z["W"]), int(z["T"]),
                             float(z["dx"]), float(z["dy"]), float(z["dt"]),
                             z["u"], z["v"])
        cfg = vfcp.Config(predictor=str(z["predictor"]),
                          radius=int(z["radius"]), bx=int(z["bx"]),
                          by=int(z["by"]), stride=int(z["stride"]),
                          lam=float(z["lam"]), theta=float(z["theta"]),
                          d_max=float(z["d_max"]), n_max=int(z["n_max"]),
                          stats=True)
        a = vfcp.compress(f, float(z["eps"]), cfg, relative=bool(z["relative"]))
        s = a.stats
        out[f"{name}__symbols"] = np.asarray(s.symbols, np.int32)
        out[f"{name}__signed"] = np.asarray(s.signed_indices, np.int32)
        out[f"{name}__overflow"] = np.int64(s.overflow_count)
        out[f"{name}__lossless"] = np.int64(s.lossless_vertices)
        out[f"{name}__modes"] = np.asarray(s.modes, np.uint8)
        out[f"{name}__faces"] = np.int64(s.critical_faces)
        print(name, s.overflow_count, s.lossless_vertices, s.critical_faces,
              s.modes.shape)
    np.savez_compressed(GOLDEN / "compress_stats.npz", **out)


if __name__ == "__main__":
    main()
