"""Stage times of the public compress() on config 5 (steady state)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, huffman, synth  # noqa: E402

H, W, T, u, v = synth.generate(5, 8192, 8192, 16)
up = torch.from_numpy(u).pin_memory()
vp = torch.from_numpy(v).pin_memory()
fh = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, up, vp)
cfg = vg.Config(backend="identity")


def tm(fn, label):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    print(f"{label}: {time.perf_counter() - t0:.3f} s", flush=True)
    return r


for it in range(2):
    print("-- iteration", it)
    s = tm(lambda: codec.compress_device(fh, 1e-3, cfg, relative=True), "compress_device (H2D + kernels)")
    tm(lambda: huffman.encode_device(s.codes, 32), "encode_device codes")
    tm(lambda: huffman.encode_device(s.qd, 2 * cfg.radius, cfg.radius - 4096), "encode_device qd")
    tm(lambda: (s.ld.cpu(), s.ll.cpu(), s.modes.cpu()), "small streams to host")
    del s
    a = tm(lambda: vg.compress(fh, 1e-3, cfg, relative=True), "compress()")
    del a
