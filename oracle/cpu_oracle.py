"""CPU ORACLE driver -- test infrastructure, NOT product code.

Drives the plain-C restatement in vfcp_oracle.c (ctypes) with the
reference's own orchestration (codec.py:321-398 compress, codec.py:401-453
decompress) to produce the reference's symbol streams:

    codes (u8[N]), l_d (bool[N]), modes (u8[T-1,nby,nbx]), qd (int32),
    ll (int64), recon fixed (int64[T,H,W]), plus the critical-face mask.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this module.  Parity of this oracle with the
reference itself is pinned by tests/test_oracle_golden.py against
tests/golden/*.npz, which oracle/gen_golden.py produced by running the real
reference (/root/reference/pkg/src/vfcp) in the build container.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "liboracle.so"
_lib = None

FIXED_LIMIT = 1 << 30
CODE_LOSSLESS = 31
K_MAX = 30

_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(dtype=np.uint8, flags="C_CONTIGUOUS")
_u16p = np.ctypeslib.ndpointer(dtype=np.uint16, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_I64 = ctypes.c_int64
_I = ctypes.c_int
_D = ctypes.c_double
_P = ctypes.c_void_p


def build() -> Path:
    """Compile oracle/_build/liboracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.or_to_fixed.restype = _I64
        L.or_to_fixed.argtypes = [_P, _I, _I64, _D, _i32p]
        L.or_range.restype = None
        L.or_range.argtypes = [_P, _P, _I, _I64, _f64p]
        L.or_analyze.restype = None
        L.or_analyze.argtypes = [_I, _I, _I, _i32p, _i32p, _I64, _P, _P]
        L.or_quantize_eb.restype = _I
        L.or_quantize_eb.argtypes = [_I64, _I64]
        L.or_codes.restype = None
        L.or_codes.argtypes = [_i64p, _I64, _I64, _u8p, _u8p]
        L.or_face_positive.restype = _I
        L.or_face_positive.argtypes = [_I64] * 9
        L.or_sos_sign.restype = _I
        L.or_sos_sign.argtypes = [_I64] * 9
        L.or_edge_eb.restype = _I64
        L.or_edge_eb.argtypes = [_I64] * 4
        L.or_face_eb.restype = _I64
        L.or_face_eb.argtypes = [_I64] * 6
        L.or_rha.restype = _I64
        L.or_rha.argtypes = [_D]
        L.or_bilinear.restype = _I64
        L.or_bilinear.argtypes = [_i64p, _I, _I, _D, _D]
        L.or_sl_departure.restype = None
        L.or_sl_departure.argtypes = [_i64p, _i64p, _I, _I, _I, _I, _D, _D,
                                      _D, _I64, _f64p]
        L.or_score_frame.restype = None
        L.or_score_frame.argtypes = [
            _I, _I, _i64p, _i64p, _i64p, _i64p, _I64, _I64, _I, _I, _I, _D,
            _D, _D, _D, _D, _D, _I64, _u8p, _f64p]
        L.or_encode_frame.restype = None
        L.or_encode_frame.argtypes = [
            _I, _I, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _i64p, _u8p,
            _I, _I, _I, _D, _D, _D, _I64, _I64, _i32p,
            ctypes.POINTER(_I64), _i64p, ctypes.POINTER(_I64)]
        L.or_decode_frame.restype = None
        L.or_decode_frame.argtypes = [
            _I, _I, _i64p, _i64p, _i64p, _i64p, _i64p, _u8p, _I, _I, _I, _D,
            _D, _D, _I64, _I64, _i32p, ctypes.POINTER(_I64), _i64p,
            ctypes.POINTER(_I64)]
        _lib = L
    return _lib


# --------------------------------------------------------------------------
# host-side scalar helpers restated from the reference

def choose_scale(max_abs: float) -> float:
    """field.py:300-310."""
    if max_abs == 0.0:
        return float(FIXED_LIMIT)
    k = int(math.floor(math.log2(FIXED_LIMIT / max_abs)))
    s = 2.0 ** k
    while max_abs * s >= FIXED_LIMIT:
        s /= 2.0
    while max_abs * (s * 2.0) < FIXED_LIMIT:
        s *= 2.0
    return s


def tau_from_eps(eps: float, scale: float) -> int:
    """codec.py:71-77."""
    return max(0, int(math.floor(eps * scale - 0.5)))


def quantize_eb(xi: int, tau: int) -> int:
    return int(lib().or_quantize_eb(int(xi), int(tau)))


def value_range(u, v) -> float:
    """field.py:69-73."""
    lo = min(float(u.min()), float(v.min()))
    hi = max(float(u.max()), float(v.max()))
    return hi - lo


def _dtype_code(a):
    if a.dtype == np.float32:
        return 0
    if a.dtype == np.float64:
        return 1
    raise TypeError(a.dtype)


def to_fixed(u, v, scale: float | None = None):
    """field.py:313-336 -> (u_fp int32, v_fp int32, S)."""
    u = np.ascontiguousarray(u)
    v = np.ascontiguousarray(v)
    n = u.size
    L = lib()
    uo = np.empty(n, np.int32)
    vo = np.empty(n, np.int32)
    if scale is None:
        m64 = max(float(np.abs(u.astype(np.float64)).max()),
                  float(np.abs(v.astype(np.float64)).max()))
        s = choose_scale(m64)
        while True:
            m = max(L.or_to_fixed(u.ctypes.data, _dtype_code(u), n, s, uo),
                    L.or_to_fixed(v.ctypes.data, _dtype_code(v), n, s, vo))
            if m < FIXED_LIMIT:
                break
            s /= 2.0
    else:
        s = float(scale)
        L.or_to_fixed(u.ctypes.data, _dtype_code(u), n, s, uo)
        L.or_to_fixed(v.ctypes.data, _dtype_code(v), n, s, vo)
    return uo, vo, s


def analyze(H, W, T, u_fp, v_fp, tau, want_mask=True, want_xi=True):
    """predicates.build_critical_face_set + ebounds.derive_all.

    Returns (mask u16[N] or None, xi i64[N] or None)."""
    n = H * W * T
    mask = np.zeros(n, np.uint16) if want_mask else None
    xi = np.zeros(n, np.int64) if want_xi else None
    lib().or_analyze(H, W, T, np.ascontiguousarray(u_fp, np.int32),
                     np.ascontiguousarray(v_fp, np.int32), int(tau),
                     mask.ctypes.data if mask is not None else None,
                     xi.ctypes.data if xi is not None else None)
    return mask, xi


def codes_from_xi(xi, tau):
    n = xi.size
    codes = np.empty(n, np.uint8)
    ld = np.empty(n, np.uint8)
    lib().or_codes(np.ascontiguousarray(xi, np.int64), n, int(tau), codes, ld)
    return codes, ld.astype(bool)


FACE_CLASS_NAMES = ("slice_lower", "slice_upper", "wall_h1", "wall_h2",
                    "wall_v1", "wall_v2", "wall_d1", "wall_d2",
                    "int_lower_a", "int_lower_b", "int_upper_a",
                    "int_upper_b")
# (dt, di, dj) of (a, b, c) from the anchor, mesh.py:100-128
FACE_CLASS_OFFSETS = (
    ((0, 0, 0), (0, 1, 0), (0, 1, 1)),
    ((0, 0, 0), (0, 0, 1), (0, 1, 1)),
    ((0, 0, 0), (0, 0, 1), (1, 0, 1)),
    ((0, 0, 0), (1, 0, 0), (1, 0, 1)),
    ((0, 0, 0), (0, 1, 0), (1, 1, 0)),
    ((0, 0, 0), (1, 0, 0), (1, 1, 0)),
    ((0, 0, 0), (0, 1, 1), (1, 1, 1)),
    ((0, 0, 0), (1, 0, 0), (1, 1, 1)),
    ((0, 0, 0), (0, 1, 0), (1, 1, 1)),
    ((0, 0, 0), (1, 1, 0), (1, 1, 1)),
    ((0, 0, 0), (0, 0, 1), (1, 1, 1)),
    ((0, 0, 0), (1, 0, 1), (1, 1, 1)),
)


def mask_to_faces(mask, H, W, T):
    """12-bit anchor mask -> (slice set, slab set) of sorted id triples."""
    hw = H * W
    sl, sb = set(), set()
    anchors = np.flatnonzero(mask)
    for an in anchors.tolist():
        m = int(mask[an])
        for c in range(12):
            if m >> c & 1:
                tri = tuple(an + dt * hw + di * W + dj
                            for dt, di, dj in FACE_CLASS_OFFSETS[c])
                (sl if c < 2 else sb).add(tri)
    return frozenset(sl), frozenset(sb)


def faces_to_mask(slice_faces, slab_faces, H, W, T):
    """Inverse of mask_to_faces using the unique class signatures."""
    hw = H * W
    sig = {}
    for c, offs in enumerate(FACE_CLASS_OFFSETS):
        o = [dt * hw + di * W + dj for dt, di, dj in offs]
        sig[(o[1] - o[0], o[2] - o[0])] = c
    mask = np.zeros(H * W * T, np.uint16)
    for a, b, c in list(slice_faces) + list(slab_faces):
        mask[a] |= 1 << sig[(b - a, c - a)]
    return mask


# --------------------------------------------------------------------------
# orchestration: codec.py:321-398 compress (symbol streams, no entropy stage)

def _cfl(dx, dy, dt, scale):
    """predictors.py:117-119."""
    return (dt / dx) / scale, (dt / dy) / scale


def compress_streams(u, v, H, W, T, dx, dy, dt, eps, cfg, relative=False,
                     want_mask=False):
    """Everything codec.compress computes before huffman/zlib.

    cfg: object with predictor, bx, by, stride, lam, theta, radius, d_max,
    n_max (reference Config or the product Config)."""
    if eps < 0:
        raise ValueError("eps must be non-negative")
    u = np.ascontiguousarray(u)
    v = np.ascontiguousarray(v)
    if relative:
        eps = eps * value_range(u, v)
    uf, vf, S = to_fixed(u, v)
    tau = tau_from_eps(eps, S)
    mask, xi = analyze(H, W, T, uf, vf, tau, want_mask=want_mask)
    codes, ld = codes_from_xi(xi, tau)
    eq = np.where(codes == CODE_LOSSLESS, 0,
                  tau >> np.minimum(codes, K_MAX).astype(np.int64)).astype(np.int64)
    uo3 = uf.astype(np.int64).reshape(T, H, W)
    vo3 = vf.astype(np.int64).reshape(T, H, W)
    eq3 = eq.reshape(T, H, W)
    cfl_x, cfl_y = _cfl(dx, dy, dt, S)
    nby, nbx = -(-H // cfg.by), -(-W // cfg.bx)
    n = H * W * T
    qd = np.zeros(2 * n, np.int32)
    ll = np.zeros(2 * n, np.int64)
    qp = _I64(0)
    lp = _I64(0)
    modes_all = np.zeros((max(T - 1, 0), nby, nbx), np.uint8)
    prev_u = np.zeros((H, W), np.int64)
    prev_v = np.zeros((H, W), np.int64)
    cur_u = np.empty_like(prev_u)
    cur_v = np.empty_like(prev_v)
    recon = np.empty((2, T, H, W), np.int64)
    zero_modes = np.zeros((nby, nbx), np.uint8)
    L = lib()
    rmeta = 1.0 / (cfg.bx * cfg.by * 2)
    for t in range(T):
        if t == 0 or tau == 0 or cfg.predictor == "lorenzo":
            modes_t = zero_modes
        elif cfg.predictor == "sl":
            modes_t = np.ones((nby, nbx), np.uint8)
        else:
            modes_t = np.zeros((nby, nbx), np.uint8)
            scores = np.zeros((nby, nbx, 2), np.float64)
            L.or_score_frame(H, W, np.ascontiguousarray(uo3[t]),
                             np.ascontiguousarray(vo3[t]), prev_u, prev_v,
                             int(tau), int(cfg.radius), int(cfg.stride),
                             int(cfg.bx), int(cfg.by), float(cfg.lam), rmeta,
                             float(cfg.theta), cfl_x, cfl_y, float(cfg.d_max),
                             int(cfg.n_max), modes_t, scores)
        if t >= 1:
            modes_all[t - 1] = modes_t
        L.or_encode_frame(H, W, np.ascontiguousarray(uo3[t]),
                          np.ascontiguousarray(vo3[t]), prev_u, prev_v,
                          cur_u, cur_v, np.ascontiguousarray(eq3[t]),
                          np.ascontiguousarray(modes_t), int(t >= 1),
                          int(cfg.by), int(cfg.bx), cfl_x, cfl_y,
                          float(cfg.d_max), int(cfg.n_max), int(cfg.radius),
                          qd, ctypes.byref(qp), ll, ctypes.byref(lp))
        recon[0, t] = cur_u
        recon[1, t] = cur_v
        prev_u, cur_u = cur_u, prev_u
        prev_v, cur_v = cur_v, prev_v
    return dict(eps=eps, scale=S, tau=tau, codes=codes, ld=ld,
                xi=xi, mask=mask, modes=modes_all, qd=qd[:qp.value].copy(),
                ll=ll[:lp.value].copy(), recon=recon, u_fp=uf, v_fp=vf)


def decompress_streams(H, W, T, dx, dy, dt, scale, tau, cfg, codes, qd, ll,
                       modes):
    """codec.py:401-453 minus the entropy stage -> recon fixed (2,T,H,W)."""
    eq = np.where(codes == CODE_LOSSLESS, 0,
                  tau >> np.minimum(codes, K_MAX).astype(np.int64)).astype(np.int64)
    eq3 = eq.reshape(T, H, W)
    cfl_x, cfl_y = _cfl(dx, dy, dt, scale)
    nby, nbx = -(-H // cfg.by), -(-W // cfg.bx)
    prev_u = np.zeros((H, W), np.int64)
    prev_v = np.zeros((H, W), np.int64)
    cur_u = np.empty_like(prev_u)
    cur_v = np.empty_like(prev_v)
    zero_modes = np.zeros((nby, nbx), np.uint8)
    qd = np.ascontiguousarray(qd, np.int32)
    ll = np.ascontiguousarray(ll, np.int64)
    qp = _I64(0)
    lp = _I64(0)
    out = np.empty((2, T, H, W), np.int64)
    L = lib()
    for t in range(T):
        m = np.ascontiguousarray(modes[t - 1]) if t >= 1 else zero_modes
        L.or_decode_frame(H, W, prev_u, prev_v, cur_u, cur_v,
                          np.ascontiguousarray(eq3[t]), m, int(t >= 1),
                          int(cfg.by), int(cfg.bx), cfl_x, cfl_y,
                          float(cfg.d_max), int(cfg.n_max), int(cfg.radius),
                          qd, ctypes.byref(qp), ll, ctypes.byref(lp))
        out[0, t] = cur_u
        out[1, t] = cur_v
        prev_u, cur_u = cur_u, prev_u
        prev_v, cur_v = cur_v, prev_v
    if qp.value != qd.size:
        raise ValueError("residual stream length mismatch")
    if lp.value != ll.size:
        raise ValueError("lossless stream length mismatch")
    return out
