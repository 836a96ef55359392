"""World-size-2 host logic of the replica path on CPU/gloo.

Each rank compresses its own small field with the host-side stages that the
GPU path shares (CPU oracle streams -> Huffman -> Archive bytes) and the
timing reduction is the max over ranks; the per-rank archives must equal
the single-process ones (replicas are independent)."""

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _archive_bytes(rank):
    from oracle import cpu_oracle as O
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200 import synth, huffman, codec
    H, W, T, u, v = synth.generate(1, 24, 40, 3 + rank)
    cfg = vg.Config()
    r = O.compress_streams(u, v, H, W, T, 1.0, 1.0, 1.0, 1e-2, cfg, relative=True)
    a = codec.Archive(H, W, T, 1.0, 1.0, 1.0, r["scale"], r["eps"], r["tau"], cfg,
                      huffman.encode(r["codes"].reshape(-1), 32),
                      huffman.encode(r["qd"].astype(np.uint16), 2 * cfg.radius),
                      np.packbits(r["ld"].reshape(-1)).tobytes(),
                      r["ll"].astype("<i8").tobytes(),
                      np.packbits(r["modes"].reshape(-1)).tobytes())
    return a.to_bytes()


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2510_25143_b200 import replicas
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blob = _archive_bytes(rank)
        replicas.barrier(dist, cuda=False)
        t_max = replicas.max_over_ranks(1.0 + rank, dist, device="cpu")
        total = replicas.sum_over_ranks(float(len(blob)), dist, device="cpu")
        q.put((rank, blob, t_max, total))
    finally:
        dist.destroy_process_group()


def test_replicas_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    blobs = [r[1] for r in res]
    assert all(r[2] == 2.0 for r in res)               # max over ranks
    assert all(r[3] == float(sum(map(len, blobs))) for r in res)
    for rank, blob in enumerate(blobs):                 # replicas independent
        assert blob == _archive_bytes(rank)


# ---------------------------------------------- row bands (bands.py, §8e)

def _band_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                      RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2510_25143_b200 import bands, synth
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        H, W, T, u, v = synth.generate(1, 37, 20, 3)
        r0, r1 = bands.band_rows(H, rank, world)
        h0, h1 = bands.halo_rows(H, r0, r1)
        ub = u.reshape(T, H, W)[:, r0:r1].astype(np.float64)
        vb = v.reshape(T, H, W)[:, r0:r1].astype(np.float64)
        # the band's own (min, max, max|x|) -- on the device in the product
        # path (vfcp_value_range); numpy stands in here
        lo = float(min(ub.min(), vb.min()))
        hi = float(max(ub.max(), vb.max()))
        ma = float(max(np.abs(ub).max(), np.abs(vb).max()))
        eps, S = bands.band_scale(lo, hi, ma, 1e-2, True, dist, device="cpu")
        fc = bands.sum_counts((3 + rank, 10 * rank), dist, device="cpu")
        q.put((rank, (r0, r1, h0, h1), eps, S, fc))
    finally:
        dist.destroy_process_group()


def test_bands_gloo_world2():
    import torch.multiprocessing as mp
    from paper_2510_25143_b200 import bands, synth
    from paper_2510_25143_b200.field import scale_for
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_band_worker, args=(r, 2, port, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    H, W, T, u, v = synth.generate(1, 37, 20, 3)
    x = np.concatenate([u, v]).astype(np.float64)
    eps = 1e-2 * (float(x.max()) - float(x.min()))
    S = scale_for(float(np.abs(x).max()))
    assert [r[1][:2] for r in res] == [(0, 19), (19, 37)]
    assert [r[1][2:] for r in res] == [(0, 20), (18, 37)]
    assert all(r[2] == eps and r[3] == S for r in res)
    assert all(r[4] == (7, 10) for r in res)          # fc_t, fc_s summed


def test_band_rows_partition():
    from paper_2510_25143_b200 import bands
    for H in (2, 7, 64, 8192):
        for world in (1, 2, 3, 8):
            rows = [bands.band_rows(H, r, world) for r in range(world)]
            assert rows[0][0] == 0 and rows[-1][1] == H
            assert all(a[1] == b[0] for a, b in zip(rows, rows[1:]))
            sizes = [b - a for a, b in rows]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        bands.band_rows(8, 2, 2)
