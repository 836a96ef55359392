import sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from conftest import load_golden
import paper_2510_25143_b200 as vg
name = sys.argv[1] if len(sys.argv) > 1 else 'vortex_small'
g = load_golden(name)
b = vg.Archive.from_bytes(bytes(g['archive']))
r = vg.reconstruct_fixed(b)
print(name, np.array_equal(r.u_fp, g['recon'][0]), np.array_equal(r.v_fp, g['recon'][1]))
