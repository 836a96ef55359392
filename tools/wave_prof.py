"""Per-phase cycle breakdown of the wavefront kernels (VFCP_WAVE_PROFILE)."""
import os, sys, time
if not os.environ.get("NOPROF"): os.environ.setdefault("VFCP_WAVE_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2510_25143_b200 as vg
from paper_2510_25143_b200 import synth, codec
cfgid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
H, W, T = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (None, None, None)
H, W, T, u, v = synth.generate(cfgid, H, W, T)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
cfg = vg.Config(predictor=os.environ.get("PRED", "mop"))
eps = float(os.environ.get("EPS", "1e-3"))
from paper_2510_25143_b200 import _lib
s = vg.compress_device(f, eps, cfg, relative=True)
_lib.prof_enable(True)
torch.cuda.synchronize(); t0 = time.perf_counter()
s = vg.compress_device(f, eps, cfg, relative=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t0
pr = _lib.prof_collect(); _lib.prof_enable(False)
print("compress s", round(dt, 4), {k: round(v[0], 3) for k, v in pr.items() if v[1]}, flush=True)
print("sl frac", float(s.modes.float().mean()) if s.modes.numel() else 0)
a = codec.Archive(H, W, T, 1.0, 1.0, 1.0, s.scale, s.eps, s.tau, cfg, b"", b"", s.ld.cpu().numpy().tobytes(), b"", b"")
kw = dict(codes=s.codes, qd=s.qd, ll=s.ll, modes=s.modes, ld=s.ld)
from paper_2510_25143_b200 import _lib
for _ in range(3):
    _lib.prof_enable(True)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    vg.decompress_device(a, **kw)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    pr = _lib.prof_collect(); _lib.prof_enable(False)
    print("decode s", round(dt, 4), {k: round(v[0], 3) for k, v in pr.items() if v[1]}, flush=True)
