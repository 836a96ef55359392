import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import load_golden
import paper_2510_25143_b200 as vg
name = sys.argv[1]
g = load_golden(name)
H, W, T = int(g['H']), int(g['W']), int(g['T'])
f = vg.FieldSeries(H, W, T, float(g['dx']), float(g['dy']), float(g['dt']), g['u'], g['v'])
cfg = vg.Config(predictor=str(g['predictor']), radius=int(g['radius']))
s = vg.compress_device(f, float(g['eps']), cfg, relative=bool(g['relative']))
print('tau', s.tau, 'modes equal', np.array_equal(s.modes.cpu().numpy(), g['modes'].reshape(-1)))
qd = s.qd.cpu().numpy().astype(np.int64); ref = g['qd'].astype(np.int64)
codes = g['codes']; nl = codes != 31
pos = np.cumsum(nl) - 1   # symbol pair index per vertex
bad = np.flatnonzero(qd != ref)
print('n bad', bad.size, 'of', ref.size)
if bad.size:
    k = bad[0] // 2
    v = np.flatnonzero(nl)[k]
    t, r = divmod(v, H * W); i, j = divmod(r, W)
    print('first bad vertex t,i,j', t, i, j, 'comp', bad[0] % 2, 'got', qd[bad[0]], 'want', ref[bad[0]])
    nby, nbx = -(-H // 32), -(-W // 32)
    if t >= 1: print('mode of block', g['modes'][t-1][i // 32][j // 32])
    # count bad by frame
    vb = np.flatnonzero(nl)[bad // 2]
    print('bad per frame', np.bincount(vb // (H * W), minlength=T))
