"""Phases of compress() -> Archive after the frame-streamed compress_device
(config 5, pinned host input)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, huffman, synth  # noqa: E402

H, W, T, u, v = synth.generate(5, None, None, None)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).pin_memory(),
                   torch.from_numpy(v).pin_memory())
cfg = vg.Config(backend="identity")
for _ in range(3):
    vg.compress(f, 1e-3, cfg, relative=True)
for rep in range(3):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    s = codec.compress_device(f, 1e-3, cfg, relative=True, want_hist=True)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    pend = huffman.encode_device_many([
        (s.qd, 2 * cfg.radius, max(0, cfg.radius - 4096), s.hist["qd"]),
        (s.codes, 32, 0, s.hist["codes"])])
    t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    b0 = pend[0].result(); t.append(time.perf_counter())
    b1 = pend[1].result(); t.append(time.perf_counter())
    d = [1e3 * (t[i + 1] - t[i]) for i in range(len(t) - 1)]
    print(f"compress_device {d[0]:.1f} | encode_device_many enqueue {d[1]:.1f} | "
          f"device pack + D2H done {d[2]:.1f} | qd bytes {d[3]:.1f} | codes bytes {d[4]:.1f} ms"
          f"  ({len(b0) / 1e6:.0f} + {len(b1) / 1e6:.0f} MB)", flush=True)
    del s, pend, b0, b1
import os  # noqa: E402
os.environ["VFCP_ARCHIVE_TIMES"] = "1"
for _ in range(3):
    t0 = time.perf_counter()
    a = vg.compress(f, 1e-3, cfg, relative=True)
    t1 = time.perf_counter()
    del a
    t2 = time.perf_counter()
    print(f"compress() {1e3 * (t1 - t0):.1f} ms, freeing the archive {1e3 * (t2 - t1):.1f} ms", flush=True)
