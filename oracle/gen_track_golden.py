"""Generate tests/golden/track_*.npz by running the REAL reference's
trajectory extraction (tracking.py:75-141, crossing points
predicates.py:304-318) on the input fields of the existing field fixtures.

Test infrastructure (not product code).  Run here, where /root/reference is
mounted; the GPU box only reads the fixtures:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/vfcp_numba python oracle/gen_track_golden.py

Each fixture holds the source fixture's name, the components as a flat face
list (`faces` [n, 3], `comp` [n] component id per face in chain order,
`loop` [n_comp]), the crossing points `xyt` [n, 3] and the CSV text the
reference's write_trajectory_csv produced.
"""

from __future__ import annotations

import sys
import tempfile
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[0] = str(ROOT)

import vfcp  # noqa: E402  (the reference, via PYTHONPATH)
from vfcp import tracking  # noqa: E402

GOLD = ROOT / "tests" / "golden"


def main():
    n = 0
    for src in sorted(GOLD.glob("field_*.npz")):
        z = np.load(src)
        if int(z["n_faces"]) == 0 or z["u"].size > 200_000:
            continue
        f = vfcp.FieldSeries(int(z["H"]), int(z["W"]), int(z["T"]),
                             float(z["dx"]), float(z["dy"]), float(z["dt"]),
                             z["u"], z["v"])
        try:
            g = tracking.extract_trajectories(vfcp.to_fixed(f), f.dx, f.dy, f.dt)
        except tracking.TopologyError as err:
            print(src.name, "TopologyError", err)
            continue
        faces, comp, xyt = [], [], []
        for k, chain in enumerate(g.components):
            for fk in chain:
                faces.append(fk)
                comp.append(k)
                xyt.append(g.nodes[fk])
        with tempfile.TemporaryDirectory() as d:
            p = Path(d) / "t.csv"
            tracking.write_trajectory_csv(g, p)
            text = p.read_text()
        out = GOLD / ("track_" + src.name[len("field_"):])
        np.savez_compressed(
            out, source=src.name,
            faces=np.asarray(faces, np.int64).reshape(-1, 3),
            comp=np.asarray(comp, np.int64),
            loop=np.asarray(g.loops, np.bool_),
            xyt=np.asarray(xyt, np.float64).reshape(-1, 3),
            csv=text)
        n += 1
        print(out.name, len(g.components), "components", len(faces), "faces",
              sum(g.loops), "loops")
    print(n, "fixtures")


if __name__ == "__main__":
    main()
