"""Device Huffman encode/decode of a synthetic residual stream (2^31 u16
symbols, geometric around the radius) -- per-kernel times under ncu."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_25143_b200 import huffman  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 31)
g = torch.Generator(device="cuda").manual_seed(0)
x = torch.empty(n, dtype=torch.float32, device="cuda").exponential_(1.0, generator=g)
sgn = torch.randint(0, 2, (n,), device="cuda", generator=g) * 2 - 1
sym = (32768 + (x * 0.8).floor().to(torch.int32) * sgn).clamp(1, 65535).to(torch.int32).to(torch.uint16)
del x, sgn
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    blob = huffman.encode_device(sym, 65536, 32768 - 4096)
    t1 = time.perf_counter()
    out = huffman.decode_device(blob, np.uint16)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"encode {t1 - t0:.3f} s ({len(blob) / 1e6:.0f} MB), decode {t2 - t1:.3f} s, "
          f"equal {bool((out == sym).all().item())}", flush=True)
