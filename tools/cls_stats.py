"""Block classes per frame (VFCP_CLS_STATS, stderr): how many blocks of each
frame are REG / KNOWN / swept by the chain.
    python tools/cls_stats.py [config] [T] [eps]"""
import os
import sys
from pathlib import Path

os.environ["VFCP_CLS_STATS"] = "1"
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
s = codec.compress_device(f, eps, vg.Config(), relative=True)
torch.cuda.synchronize()
print("tau", s.tau, "scale", s.scale)
