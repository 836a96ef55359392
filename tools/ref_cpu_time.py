"""Time the REAL reference (vfcp, Python + numba, single-threaded) on the
BASELINE configs in the build container, for the CPU baseline labels of the
measurement matrix (the reference cannot travel to the GPU box).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/vfcp_numba \
        python tools/ref_cpu_time.py > profiles/ref_cpu_numba_r02.json

Configs 1-3 at full size; configs 4 and 5 at a reduced frame count (the
stock reference needs ~240 B/vertex of host memory).
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(1, str(ROOT))
import vfcp  # noqa: E402  (the reference)

from paper_2510_25143_b200 import synth  # noqa: E402

RUNS = [(1, 1e-2, None, None, None), (2, 1e-3, None, None, None),
        (3, 1e-2, None, None, None), (3, 1e-3, None, None, None),
        (4, 1e-3, None, None, 4), (5, 1e-3, 2048, 2048, 4)]


def main():
    # JIT warm-up on a tiny field
    H, W, T, u, v = synth.generate(1, 16, 16, 4)
    f = vfcp.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    vfcp.decompress(vfcp.Archive.from_bytes(vfcp.compress(f, 1e-2, relative=True).to_bytes()))
    out = {"what": "reference vfcp (numba, 1 thread) timed with perf_counter in "
                   "the build container: compress(...).to_bytes() and "
                   "decompress(Archive.from_bytes(blob))",
           "host": f"{os.cpu_count()} cores (1 used)", "runs": []}
    for cfg, eps, Hs, Ws, Ts in RUNS:
        H, W, T, u, v = synth.generate(cfg, Hs, Ws, Ts)
        f = vfcp.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
        t0 = time.perf_counter()
        blob = vfcp.compress(f, eps, relative=True).to_bytes()
        tc = time.perf_counter() - t0
        t0 = time.perf_counter()
        vfcp.decompress(vfcp.Archive.from_bytes(blob))
        td = time.perf_counter() - t0
        mb = 8.0 * H * W * T / 1e6
        r = {"config": cfg, "eps_rel": eps, "H": H, "W": W, "T": T,
             "compress_s": round(tc, 2), "decompress_s": round(td, 2),
             "compress_MBps": round(mb / tc, 2),
             "decompress_MBps": round(mb / td, 2),
             "full_size": Hs is None and Ts is None}
        out["runs"].append(r)
        print(json.dumps(r), file=sys.stderr, flush=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
