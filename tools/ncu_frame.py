"""One compress + decompress of a config at a few frames, for ncu captures
of single kernels (e.g. -k regex:enc_block --launch-skip 1 -c 1).

    python tools/ncu_frame.py [config] [T] [eps]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, synth  # noqa: E402

cfg_id = int(sys.argv[1]) if len(sys.argv) > 1 else 5
T = int(sys.argv[2]) if len(sys.argv) > 2 else 3
eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-3
H, W, T, u, v = synth.generate(cfg_id, None, None, T)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).cuda(),
                   torch.from_numpy(v).cuda())
cfg = vg.Config()
s = codec.compress_device(f, eps, cfg, relative=True)
a_meta = codec.Archive(H, W, T, 1.0, 1.0, 1.0, s.scale, s.eps, s.tau, cfg,
                       b"", b"", s.ld.cpu().numpy().tobytes(), b"", b"")
out = vg.decompress_device(a_meta, codes=s.codes, qd=s.qd, ll=s.ll,
                           modes=s.modes, ld=s.ld)
torch.cuda.synchronize()
print("ok", H, W, T)
