"""decompress(Archive) -> float64 host arrays on config 5: the call and its
pieces (section H2D + Huffman decode, frame loop with per-frame D2H)."""
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
arc = vg.compress(f, 1e-3, vg.Config(), relative=True)
gb = 8.0 * H * W * T / 1e9


def t_of(fn, n=3, warm=2):
    for _ in range(warm):
        r = None
        r = fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        r = None
        r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n


d = t_of(lambda: vg.decompress(arc))
print(f"decompress(): {1e3 * d:.1f} ms ({gb / d:.2f} GB/s of fp32 field; "
      f"D2H {16 * H * W * T / 1e9:.1f} GB = {16 * H * W * T / d / 1e9:.1f} GB/s)")
d = t_of(lambda: huffman.decode_device(arc.q_d, np.uint16))
print(f"q_d section -> device symbols: {1e3 * d:.1f} ms")
d = t_of(lambda: huffman.decode_device(arc.q_xi, np.uint8))
print(f"q_xi section -> device codes: {1e3 * d:.1f} ms")
d = t_of(lambda: codec.decompress_device(arc))
print(f"decompress_device (output stays on the device): {1e3 * d:.1f} ms")
hu = torch.empty(H * W * T, dtype=torch.float64, pin_memory=True)
hv = torch.empty(H * W * T, dtype=torch.float64, pin_memory=True)
d = t_of(lambda: codec.decompress_device(arc, host_out=(hu, hv)))
print(f"decompress_device(host_out): {1e3 * d:.1f} ms")
du = torch.empty(H * W * T, dtype=torch.float64, device="cuda")
d = t_of(lambda: (hu.copy_(du, non_blocking=True), hv.copy_(du, non_blocking=True)))
print(f"D2H of 2 x {du.numel() * 8 / 1e9:.1f} GB alone: {1e3 * d:.1f} ms")
