import sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2510_25143_b200 as vg
from paper_2510_25143_b200 import synth, codec, huffman
H, W, T, u, v = synth.generate(5, 8192, 8192, 16)
f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda())
cfg = vg.Config(backend="identity")
a = vg.compress(f, 1e-3, cfg, relative=True)
b = vg.Archive.from_bytes(a.to_bytes())
def tm(fn, label):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = fn(); torch.cuda.synchronize(); print(f"{label}: {time.perf_counter()-t0:.3f} s", flush=True); return r
for it in range(2):
    tm(lambda: huffman.decode_device(b.q_xi, np.uint8), "decode q_xi")
    tm(lambda: huffman.decode_device(b.q_d, np.uint16), "decode q_d")
    out = tm(lambda: codec.decompress_device(b), "decompress_device")
    tm(lambda: (codec._to_host(out[0]), codec._to_host(out[1])), "D2H pinned")
    tm(lambda: (out[0].cpu(), out[1].cpu()), "D2H pageable")
    tm(lambda: vg.decompress(b), "decompress()")
