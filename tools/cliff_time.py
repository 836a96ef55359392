"""Where the block kernels stop: config 5 (8192 x 8192 x 16) timed on the
generic int64 kernels (encode.cu / decode.cu) that take every configuration
the block path does not -- forced with VFCP_SLOW_PATH, radius 65536 (17-bit
symbols) and eps_rel 0.6 (tau' >= 2^29) -- next to the block path at the
same settings where it applies (eps_rel 0.2: tau' in [2^28, 2^29), which
round 1 sent to the generic kernels).

    python tools/cliff_time.py > profiles/cliff_r02.json
"""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, synth  # noqa: E402


def timed(f, eps, cfg, slow=False, steps=2):
    if slow:
        os.environ["VFCP_SLOW_PATH"] = "1"
    try:
        s = codec.compress_device(f, eps, cfg, relative=True)   # warm-up
        am = codec.Archive(f.H, f.W, f.T, 1.0, 1.0, 1.0, s.scale, s.eps,
                           s.tau, cfg, b"", b"", s.ld.cpu().numpy().tobytes(),
                           b"", b"")
        kw = dict(codes=s.codes, qd=s.qd, ll=s.ll, modes=s.modes, ld=s.ld)
        out = vg.decompress_device(am, **kw)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(steps):
            s2 = codec.compress_device(f, eps, cfg, relative=True)
        torch.cuda.synchronize()
        c = (time.perf_counter() - t0) / steps
        del s2
        t0 = time.perf_counter()
        for _ in range(steps):
            out = None
            out = vg.decompress_device(am, **kw)
        torch.cuda.synchronize()
        d = (time.perf_counter() - t0) / steps
        return {"tau": int(s.tau), "compress_ms": round(c * 1e3, 1),
                "decompress_ms": round(d * 1e3, 1),
                "compress_GBps": round(8.0 * f.H * f.W * f.T / c / 1e9, 2)}
    finally:
        os.environ.pop("VFCP_SLOW_PATH", None)


def main():
    H, W, T, u, v = synth.generate(5)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).cuda(),
                       torch.from_numpy(v).cuda())
    d = vg.Config()
    rows = {
        "block path, eps_rel 1e-3": timed(f, 1e-3, d),
        "generic (VFCP_SLOW_PATH), eps_rel 1e-3": timed(f, 1e-3, d, slow=True),
        "block path, eps_rel 0.2 (tau' >= 2^28)": timed(f, 0.2, d),
        "generic, eps_rel 0.6 (tau' >= 2^29)": timed(f, 0.6, d),
        "generic, radius 65536, eps_rel 1e-3": timed(f, 1e-3, vg.Config(radius=65536)),
    }
    print(json.dumps({"what": __doc__.strip().splitlines()[0],
                      "config": "config 5, 8192x8192x16 fp32, MoP", "runs": rows},
                     indent=1))


if __name__ == "__main__":
    main()
