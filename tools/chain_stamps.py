"""Chain timing stamps of frame 1 (VFCP_CHAIN_STAMPS): per block row the
start, first-block and end times of the chain warp (stderr)."""
import os
import sys
from pathlib import Path

os.environ["VFCP_CHAIN_STAMPS"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2510_25143_b200 as vg  # noqa: E402
from paper_2510_25143_b200 import codec, synth  # noqa: E402

eps = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-3
cfg_id = int(sys.argv[2]) if len(sys.argv) > 2 else 5
H, W, T, u, v = synth.generate(cfg_id, None, None, 3)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).cuda(),
                   torch.from_numpy(v).cuda())
for _ in range(2):
    s = codec.compress_device(f, eps, vg.Config(), relative=True)
torch.cuda.synchronize()
