"""Generate tests/golden/*.npz by running the REAL reference in this container.

Test infrastructure (not product code).  Run here, where /root/reference is
mounted; the GPU box never needs the reference, only these fixtures:

    PYTHONPATH=/root/reference/pkg/src PYTHONDONTWRITEBYTECODE=1 \
    NUMBA_CACHE_DIR=/tmp/vfcp_numba python oracle/gen_golden.py

Each field fixture holds the input (float32/float64 u, v), the settings, and
the reference's outputs: scale, tau', eb codes, l_d, the critical-face set
(as a 12-bit per-anchor class mask, see oracle.FACE_CLASS_OFFSETS), modes,
qd symbols, ll, the fixed-point reconstruction and the serialized archive
(zlib and identity backends).  Primitive fixtures hold known-answer vectors
for SoS, edge/face bounds, the eb ladder, rha, bilinear and SL departure.
"""

from __future__ import annotations

import hashlib
import random
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[0] = str(ROOT)

import vfcp  # noqa: E402  (the reference, via PYTHONPATH)
from vfcp import codec, ebounds, predicates, predictors  # noqa: E402

from oracle import cpu_oracle as O  # noqa: E402
from paper_2510_25143_b200 import synth  # noqa: E402

OUT = ROOT / "tests" / "golden"


def field_case(name, f, eps, cfg, relative):
    a = vfcp.compress(f, eps, cfg, relative=relative)
    ff = vfcp.to_fixed(f)
    cfs = predicates.build_critical_face_set(ff)
    eb = ebounds.derive_all(ff, cfs, a.tau_prime)
    codes = codec._quantize_eb_vec(eb.xi, a.tau_prime)
    mask = O.faces_to_mask(cfs.slice_faces, cfs.slab_faces, f.H, f.W, f.T)
    blob = a.to_bytes()
    ident = vfcp.Archive(**{**a.__dict__, "config": vfcp.Config(
        **{**cfg.__dict__, "backend": "identity"})})
    from vfcp import huffman
    try:
        r = vfcp.reconstruct_fixed(a)
        recon = np.stack([r.u_fp, r.v_fp]).astype(np.int32)
        decode_error = ""
    except ValueError as exc:          # quirk V7 archives do not decode
        recon = np.zeros((2, 0), np.int32)
        decode_error = str(exc)
    qd = huffman.decode(a.q_d)
    ll = np.frombuffer(a.lossless_stream, dtype="<i8").astype(np.int64)
    nby, nbx = -(-f.H // cfg.by), -(-f.W // cfg.bx)
    nm = max(f.T - 1, 0) * nby * nbx
    modes = np.unpackbits(np.frombuffer(a.mode_bitmap, np.uint8))[:nm]
    rec = dict(
        H=f.H, W=f.W, T=f.T, dx=f.dx, dy=f.dy, dt=f.dt,
        u=f.u, v=f.v, eps=eps, relative=int(relative),
        eps_abs=a.eps, predictor=cfg.predictor, radius=cfg.radius,
        bx=cfg.bx, by=cfg.by, stride=cfg.stride, lam=cfg.lam,
        theta=cfg.theta, d_max=cfg.d_max, n_max=cfg.n_max,
        scale=a.scale, tau=a.tau_prime, xi=eb.xi,
        codes=codes, ld=np.packbits(eb.lossless),
        mask_anchor=np.flatnonzero(mask).astype(np.int64),
        mask_bits=mask[mask != 0],
        modes=modes.reshape(max(f.T - 1, 0), nby, nbx),
        qd=qd.astype(np.int32), ll=ll, recon=recon,
        archive=np.frombuffer(blob, np.uint8),
        archive_identity=np.frombuffer(ident.to_bytes(), np.uint8),
        archive_sha256=hashlib.sha256(blob).hexdigest(),
        decode_error=decode_error,
        n_faces=len(cfs),
    )
    np.savez_compressed(OUT / f"field_{name}.npz", **rec)
    print(f"{name}: N={f.H*f.W*f.T} faces={len(cfs)} "
          f"lossless={int(eb.lossless.sum())} sl={modes.mean() if nm else 0:.2f} "
          f"ll={ll.size} bytes={len(blob)} {decode_error}")


def quirk_v7_field():
    """4x4x2 field where one vertex gets xi = 1 with tau' = 1000: code 31 but
    l_d = 0, so the reference's own decompress raises."""
    H, W, T = 4, 4, 2
    n = H * W * T
    rng = np.random.default_rng(0)
    u = rng.uniform(100.0, 200.0, n)
    v = rng.uniform(100.0, 200.0, n)
    u[0] = 2.0 ** 20                   # pins S = 2^9
    u[5] = 2.0 / 512.0                 # fixed value 2 -> xi <= 1
    v[5] = 2.0 / 512.0
    f = vfcp.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u.astype(np.float32),
                         v.astype(np.float32))
    S = 512.0
    eps = (1000.0 + 0.75) / S          # tau' = floor(eps*S - 0.5) = 1000
    return f, eps


def integer_field(H, W, T, lim, seed):
    rng = np.random.default_rng(seed)
    n = H * W * T
    u = rng.integers(-lim, lim + 1, n).astype(np.float32)
    v = rng.integers(-lim, lim + 1, n).astype(np.float32)
    return vfcp.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)


def fields():
    C = vfcp.Config
    cases = []
    # reference fixtures (conftest.py:7-15) and constant field (:24-29)
    cases.append(("vortex_small", vfcp.gen_synthetic("moving_vortex", 16, 16, 4, seed=3), 0.01, C(), True))
    cases.append(("translation_small", vfcp.gen_synthetic("translation", 16, 16, 4, seed=3), 0.01, C(), True))
    n = 6 * 6 * 3
    cases.append(("constant", vfcp.FieldSeries(6, 6, 3, 1.0, 1.0, 1.0, np.full(n, 1.0, np.float32), np.full(n, -2.0, np.float32)), 0.01, C(), True))
    # every kind x predictor at one mid size, ragged blocks (W not /32)
    for kind in vfcp.SYNTHETIC_KINDS:
        for pred in ("mop", "lorenzo", "sl"):
            f = vfcp.gen_synthetic(kind, 40, 72, 6, seed=2)
            cases.append((f"{kind}_{pred}", f, 0.01, C(predictor=pred), True))
    # eps sweep on mop (acceptance EPS_REL) incl. tiny eps and huge eps
    f = vfcp.gen_synthetic("random_fourier", 33, 65, 5, seed=4)
    for eps in (0.001, 0.05, 0.2, 5.0):
        cases.append((f"random_fourier_eps{eps}", f, eps, C(), True))
    cases.append(("zero_eps", f, 0.0, C(), True))
    # small radius forces escapes (overflow symbols + ll stream)
    f = vfcp.gen_synthetic("vortex_pair", 32, 32, 5, seed=0)
    cases.append(("escapes_radius4", f, 0.001, C(radius=4), True))
    cases.append(("escapes_radius2_sl", f, 0.001, C(radius=2, predictor="sl"), True))
    # non-default block grid / stride / theta / substeps
    f = vfcp.gen_synthetic("translation", 48, 40, 5, seed=1, dx=0.5, dy=0.7, dt=1.3)
    cases.append(("translation_blocks", f, 0.01, C(bx=16, by=8, stride=3, theta=0.0, d_max=0.5, n_max=5), True))
    # degenerate integer data: SoS slow path everywhere
    cases.append(("int3", integer_field(12, 14, 4, 3, 5), 0.5, C(), False))
    cases.append(("int1", integer_field(9, 10, 3, 1, 6), 0.3, C(), False))
    cases.append(("int60", integer_field(10, 12, 3, 60, 7), 4.0, C(), False))
    # float64 input (recompress of a decompressed field, test_acceptance.py:276)
    f = vfcp.gen_synthetic("vortex_pair", 32, 32, 6, seed=1)
    a1 = vfcp.compress(f, 0.01, relative=True)
    r1 = vfcp.decompress(a1)
    cases.append(("recompress_f64", r1, a1.eps, C(), False))
    # quirk V7
    qf, qe = quirk_v7_field()
    cases.append(("quirk_v7", qf, qe, C(), False))
    # reduced BASELINE configs
    for cfg, shape in ((1, (64, 64, 8)), (2, (64, 80, 6)), (3, (64, 160, 6)),
                       (4, (96, 128, 4)), (5, (128, 128, 3))):
        H, W, T, u, v = synth.generate(cfg, *shape)
        fs = vfcp.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
        for eps in synth.CONFIGS[cfg]["eps"]:
            cases.append((f"cfg{cfg}_eps{eps:g}", fs, eps, C(), True))
    return cases


def primitives():
    rng = random.Random(99)
    nrng = np.random.default_rng(99)
    # SoS face predicate: generic, small-range and degenerate triples
    sos = []
    for _ in range(4000):
        lim = rng.choice([3, 6, 100, 10 ** 9 - 1])
        pts = [(rng.randint(-lim, lim), rng.randint(-lim, lim)) for _ in range(3)]
        if rng.random() < 0.3:   # force degeneracy
            k = rng.randrange(3)
            pts[k] = rng.choice([(0, 0), pts[(k + 1) % 3],
                                 (2 * pts[(k + 1) % 3][0], 2 * pts[(k + 1) % 3][1])])
        ids = sorted(rng.sample(range(10 ** 6), 3))
        res = predicates.face_has_cp_values(*pts, *ids)
        sos.append([*pts[0], *pts[1], *pts[2], *ids, int(res)])
    # orientation signs with the origin id -1
    orient = []
    for _ in range(2000):
        lim = rng.choice([2, 5, 1000])
        pts = [(rng.randint(-lim, lim), rng.randint(-lim, lim)) for _ in range(3)]
        ids = rng.sample(range(-1, 50), 3)
        orient.append([*pts[0], *pts[1], *pts[2], *ids,
                       predicates.orient2_sos(*pts, *ids)])
    # face bounds (exact L-inf) over small, medium, full ranges
    feb = []
    for _ in range(6000):
        lim = rng.choice([4, 1000, (1 << 30) - 1])
        vals = [rng.randint(-lim, lim) for _ in range(6)]
        feb.append(vals + [ebounds.face_eb_sound(*vals)])
    # eb ladder incl. boundaries (test_codec.py:23-58)
    lad = []
    for _ in range(6000):
        tau = rng.choice([rng.randint(0, 40), rng.randint(1, 1 << 24), rng.randint(1, 1 << 40)])
        k = rng.randint(0, 31)
        base = max(tau >> k, 1)
        xi = max(0, base + rng.randint(-2, 2)) if rng.random() < 0.7 else rng.randint(0, max(tau, 1) * 2)
        lad.append([xi, tau, codec.quantize_eb(xi, tau)])
    xi_arr = np.array([r[0] for r in lad], np.int64)
    vec_taus = sorted({r[1] for r in lad})[:50]
    vec = [codec._quantize_eb_vec(xi_arr, t) for t in vec_taus]
    # rha / bilinear / SL departure
    xs = np.concatenate([nrng.normal(0, 1e6, 2000), np.arange(-50, 50) + 0.5,
                         nrng.integers(-10 ** 12, 10 ** 12, 500) + 0.5])
    rha = [int(predictors._rha(float(x))) for x in xs]
    H, W = 13, 17
    frame_u = nrng.integers(-(1 << 29), 1 << 29, (H, W)).astype(np.int64)
    frame_v = nrng.integers(-(1 << 29), 1 << 29, (H, W)).astype(np.int64)
    bil_pts = nrng.uniform(-3.0, 20.0, (3000, 2))
    bil = [predictors.bilinear(frame_u, a, b) for a, b in bil_pts]
    sl = []
    for cfl in (1e-9, 3e-9, 2.0 ** -28, 1e-8):
        for i in range(H):
            for j in range(W):
                fi, fj = predictors._sl_departure(frame_u, frame_v, i, j, cfl, cfl * 0.7, 2.0, 32)
                sl.append([cfl, i, j, fi, fj])
    np.savez_compressed(
        OUT / "primitives.npz",
        sos=np.array(sos, np.int64), orient=np.array(orient, np.int64),
        face_eb=np.array(feb, np.int64), ladder=np.array(lad, np.int64),
        ladder_vec_taus=np.array(vec_taus, np.int64),
        ladder_vec=np.array(vec, np.uint8), ladder_vec_xi=xi_arr,
        rha_x=xs, rha=np.array(rha, np.int64),
        bil_frame=frame_u, bil_frame_v=frame_v, bil_pts=bil_pts,
        bil=np.array(bil, np.int64), sl=np.array(sl, np.float64),
    )
    print("primitives written")


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    primitives()
    for name, f, eps, cfg, rel in fields():
        field_case(name, f, eps, cfg, rel)


if __name__ == "__main__":
    main()
