"""Phase times of the public compress() on a config-5 workload (pinned host
input): device pipeline, device Huffman of each section, small sections.
python tools/compress_phases.py [H W T]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, huffman, synth  # noqa: E402

H, W, T = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (8192, 8192, 16)
H, W, T, u, v = synth.generate(5, H, W, T)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).pin_memory(),
                   torch.from_numpy(v).pin_memory())
cfg = vg.Config()


def tick():
    torch.cuda.synchronize()
    return time.perf_counter()


for it in range(3):
    t0 = tick()
    s = codec.compress_device(f, 1e-3, cfg, True)
    t1 = tick()
    q_xi = huffman.encode_device(s.codes, codec.EB_ALPHABET, 0)
    t2 = tick()
    q_d = huffman.encode_device(s.qd, 2 * cfg.radius, max(0, cfg.radius - 4096))
    t3 = tick()
    ld = s.ld.cpu().numpy().tobytes()
    ll = s.ll.cpu().numpy().astype("<i8").tobytes()
    mb = np.packbits(s.modes.cpu().numpy()).tobytes()
    t4 = tick()
    a = vg.compress(f, 1e-3, cfg, relative=True)
    t5 = tick()
    print(f"it {it}: compress_device {t1 - t0:.3f}  huff codes {t2 - t1:.3f} "
          f"({len(q_xi) / 1e6:.0f} MB)  huff qd {t3 - t2:.3f} ({len(q_d) / 1e6:.0f} MB)  "
          f"small {t4 - t3:.3f}  | compress() {t5 - t4:.3f}", flush=True)
    del s, a
