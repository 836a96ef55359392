"""Chain critical-path model: time per frame vs number of strips (H/32) at
fixed W, for the encoder and decoder chain kernels."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_25143_b200 as vg
from paper_2510_25143_b200 import codec, _lib
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
T = 3
rng = np.random.default_rng(0)
HS = [int(x) for x in os.environ.get('HS', '32,64,96,128,256,512,1024,2048').split(',')]
for H in HS:
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    u = np.stack([np.sin(0.01 * x + 0.02 * y + t) + 0.01 * rng.standard_normal((H, W)) for t in range(T)]).astype(np.float32)
    v = np.stack([np.cos(0.013 * x - 0.01 * y + t) + 0.01 * rng.standard_normal((H, W)) for t in range(T)]).astype(np.float32)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u.reshape(-1)).cuda(), torch.from_numpy(v.reshape(-1)).cuda())
    cfg = vg.Config()
    s = vg.compress_device(f, 1e-3, cfg, relative=True)
    _lib.prof_enable(True)
    s = vg.compress_device(f, 1e-3, cfg, relative=True)
    pe = _lib.prof_collect(); _lib.prof_enable(False)
    a = codec.Archive(H, W, T, 1.0, 1.0, 1.0, s.scale, s.eps, s.tau, cfg, b"", b"", s.ld.cpu().numpy().tobytes(), b"", b"")
    kw = dict(codes=s.codes, qd=s.qd, ll=s.ll, modes=s.modes, ld=s.ld)
    vg.decompress_device(a, **kw)
    _lib.prof_enable(True)
    vg.decompress_device(a, **kw)
    pd = _lib.prof_collect(); _lib.prof_enable(False)
    K = (H + 31) // 32
    print(f"H={H:5d} K={K:3d} enc_chain/frame={pe['encode'][0]/T*1e3:8.1f}us "
          f"dec_chain/frame={pd['decode'][0]/T*1e3:8.1f}us", flush=True)
