"""Where compress() -> Archive spends its time on config 5 (pinned host
input): the call, and the steps of the entropy stage.  (Building the codes'
Huffman section on a side stream beside the frame loop measured 296.5 ms per
call against 290.0 ms after it: the side kernels slow the block-scan chain.)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, huffman, synth  # noqa: E402

H, W, T, u, v = synth.generate(5, None, None, None)
up = torch.from_numpy(u).pin_memory()
vp = torch.from_numpy(v).pin_memory()
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, up, vp)
cfg = vg.Config(backend="identity")
gb = 8.0 * H * W * T / 1e9


def run(label, n=3):
    vg.compress(f, 1e-3, cfg, relative=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        a = vg.compress(f, 1e-3, cfg, relative=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / n
    print(f"{label}: compress() {dt * 1e3:.1f} ms  ({gb / dt:.2f} GB/s)")
    return a


run("compress()")

# steps
torch.cuda.synchronize()
t0 = time.perf_counter()
s = codec.compress_device(f, 1e-3, cfg, relative=True)
torch.cuda.synchronize()
t1 = time.perf_counter()
p = huffman.encode_device_many([(s.qd, 2 * cfg.radius, max(0, cfg.radius - 4096))])
torch.cuda.synchronize()
t2 = time.perf_counter()
b = p[0].result()
t3 = time.perf_counter()
p2 = huffman.encode_device_many([(s.codes, 32, 0)])
torch.cuda.synchronize()
t4 = time.perf_counter()
b2 = p2[0].result()
t5 = time.perf_counter()
print(f"compress_device (H2D + kernels) {1e3 * (t1 - t0):.1f} ms; qd section: "
      f"hist+lengths+pack+D2H {1e3 * (t2 - t1):.1f} ms, bytes {1e3 * (t3 - t2):.1f} ms "
      f"({len(b) / 1e6:.0f} MB); codes section: {1e3 * (t4 - t3):.1f} ms, bytes "
      f"{1e3 * (t5 - t4):.1f} ms ({len(b2) / 1e6:.0f} MB)")
