"""End-to-end compress of config 5 from page-locked host memory: the
frame-streamed path against the whole-field path (VFCP_NO_STREAM=1), and the
host range reduction alone by thread count."""
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import _lib, codec, synth  # noqa: E402

cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 5
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-3
H, W, T, u, v = synth.generate(cfgno, None, None, None)
up = torch.from_numpy(u).pin_memory()
vp = torch.from_numpy(v).pin_memory()
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, up, vp)
cfg = vg.Config()
gb = 8.0 * H * W * T / 1e9
print(f"config {cfgno}: {H}x{W}x{T}, {gb:.2f} GB, host threads {_lib.host_threads()}")

out = np.zeros(3)
for nt in (1, 4, 8, 16, 32, 64):
    t0 = time.perf_counter()
    _lib.lib().vfcp_host_range(up.data_ptr(), vp.data_ptr(), 0, up.numel(), nt,
                               out.ctypes.data)
    dt = time.perf_counter() - t0
    print(f"host range, {nt:2d} threads: {dt * 1e3:7.1f} ms  {gb / dt:6.1f} GB/s")


def run(label, fn, n=3):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = None
    for _ in range(n):
        r = None
        r = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{label}: {dt * 1e3:.1f} ms  ({gb / dt:.2f} GB/s)", flush=True)
    return r


def host_out():
    return codec.streams_to_host(vg.compress_device(f, eps, cfg, relative=True,
                                                    host_out=True))


def dev_only():
    return vg.compress_device(f, eps, cfg, relative=True)


def archive():
    return vg.compress(f, eps, vg.Config(backend="identity"), relative=True)


for nt in ("4", "8", "16"):
    os.environ["VFCP_RANGE_THREADS"] = nt
    os.environ["VFCP_STREAM_TIMES"] = "1"
    dev_only()
    os.environ.pop("VFCP_STREAM_TIMES")
    run(f"streamed, streams stay on device, {nt} range threads", dev_only)
os.environ.pop("VFCP_RANGE_THREADS")
os.environ["VFCP_STREAM_TIMES"] = "1"
host_out()
os.environ.pop("VFCP_STREAM_TIMES")
a = run("streamed, streams to host", host_out)
run("streamed, streams stay on device", dev_only)
arc = run("streamed, compress() -> Archive", archive)
os.environ["VFCP_NO_STREAM"] = "1"
b = run("whole-field, streams to host", host_out)
run("whole-field, streams stay on device", dev_only)
arc2 = run("whole-field, compress() -> Archive", archive)
for k in a:
    assert np.array_equal(a[k], b[k]), k
assert arc.to_bytes() == arc2.to_bytes()
print("streams and archive bytes equal")
