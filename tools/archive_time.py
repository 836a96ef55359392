"""Time the public compress() -> archive bytes on a config-5 workload
(device pipeline + device Huffman + host zlib) and decompress().
python tools/archive_time.py [H W T]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import synth  # noqa: E402

H, W, T = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 16)
H, W, T, u, v = synth.generate(5, H, W, T)
up = torch.from_numpy(u).pin_memory()
vp = torch.from_numpy(v).pin_memory()
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, up, vp)
for backend in ("identity", "zlib"):
    cfg = vg.Config(backend=backend)
    # warm-up (JIT, pinned host buffers of torch's caching allocator)
    w = vg.compress(f, 1e-3, cfg, relative=True)
    r = vg.decompress(vg.Archive.from_bytes(w.to_bytes()))
    del w, r
    t0 = time.perf_counter()
    a = vg.compress(f, 1e-3, cfg, relative=True)
    t1 = time.perf_counter()
    blob = a.to_bytes()
    t2 = time.perf_counter()
    b = vg.Archive.from_bytes(blob)
    t3 = time.perf_counter()
    r = vg.decompress(b)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    gb = 8.0 * H * W * T / 1e9
    print(f"{backend}: compress() {t1 - t0:.3f} s, to_bytes {t2 - t1:.3f} s "
          f"({len(blob) / 1e6:.1f} MB, CR {8.0 * H * W * T / len(blob):.1f}), "
          f"from_bytes {t3 - t2:.3f} s, decompress() {t4 - t3:.3f} s; "
          f"compress+to_bytes {gb / (t2 - t0):.2f} GB/s")
    del a, b, r, blob
