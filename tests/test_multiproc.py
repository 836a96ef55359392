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
