"""Archive codec: the reference's public compress/decompress API on a B200.

Mirrors codec.py of the reference (names, signatures, defaults, errors and
the archive byte layout, codec.py:209-293).  Everything between "field in"
and "symbol streams out" (and back) runs as sm_100a kernels through the C
ABI (include/vfcp_b200.h); the Huffman + zlib backend stays on the host as in
the reference and is timed separately.
"""

from __future__ import annotations

import ctypes
import os
import math
import struct
import time
import zlib
from dataclasses import dataclass, field as dc_field
from pathlib import Path

import numpy as np

from . import _lib, huffman
from .field import (FieldSeries, FixedField, device_range, dtype_code,
                    scale_for, to_device)

MAGIC = b"VFCP"
VERSION = 1
K_MAX = 30
CODE_LOSSLESS = 31
EB_ALPHABET = 32
FLAG_IDENTITY = 0x1
D_MAX_DEFAULT = 2.0
N_MAX_DEFAULT = 32

PREDICTORS = ("mop", "lorenzo", "sl")


@dataclass(frozen=True)
class MopConfig:
    """mop.py:26-37."""
    bx: int = 32
    by: int = 32
    stride: int = 2
    lam: float = 16.0
    theta: float = 3e-4

    @property
    def r_meta(self) -> float:
        return 1.0 / (self.bx * self.by * 2)


@dataclass(frozen=True)
class Config:
    """Single source of codec defaults (codec.py:44-68)."""
    predictor: str = "mop"        # mop | lorenzo | sl
    bx: int = 32
    by: int = 32
    stride: int = 2
    lam: float = 16.0
    theta: float = 3e-4
    radius: int = 1 << 15         # quantization index range: |idx| < radius
    d_max: float = D_MAX_DEFAULT
    n_max: int = N_MAX_DEFAULT
    backend: str = "zlib"         # zlib | identity
    stats: bool = False

    def __post_init__(self):
        if self.predictor not in PREDICTORS:
            raise ValueError(f"unknown predictor {self.predictor!r}")
        if self.backend not in ("zlib", "identity"):
            raise ValueError(f"unknown backend {self.backend!r}")

    @property
    def mop(self) -> MopConfig:
        return MopConfig(bx=self.bx, by=self.by, stride=self.stride,
                         lam=self.lam, theta=self.theta)


def tau_from_eps(eps: float, scale: float) -> int:
    """codec.py:71-77."""
    return max(0, int(math.floor(eps * scale - 0.5)))


def quantize_eb(xi: int, tau_prime: int, k_max: int = K_MAX) -> int:
    """codec.py:80-90 (scalar ladder code)."""
    if tau_prime <= 0 or xi <= 0:
        return CODE_LOSSLESS
    if xi >= tau_prime:
        return 0
    m = (tau_prime + xi - 1) // xi
    k = (m - 1).bit_length()
    if k > k_max or (tau_prime >> k) == 0:
        return CODE_LOSSLESS
    return k


def eb_from_code(code: int, tau_prime: int) -> int:
    return 0 if code == CODE_LOSSLESS else tau_prime >> code


_HEADER = struct.Struct("<4sHHIIIdddidqHHHIdddHB")


@dataclass
class Archive:
    H: int
    W: int
    T: int
    dx: float
    dy: float
    dt: float
    scale: float
    eps: float
    tau_prime: int
    config: Config
    q_xi: bytes
    q_d: bytes
    l_d: bytes
    lossless_stream: bytes
    mode_bitmap: bytes
    stats: "CompressStats | None" = dc_field(default=None, compare=False)

    @property
    def sections(self) -> tuple[bytes, ...]:
        return (self.q_xi, self.q_d, self.l_d,
                self.lossless_stream, self.mode_bitmap)

    def to_bytes(self) -> bytes:
        """codec.py:236-253."""
        cfg = self.config
        flags = FLAG_IDENTITY if cfg.backend == "identity" else 0
        scale_log2 = round(math.log2(self.scale))
        head = _HEADER.pack(
            MAGIC, VERSION, flags, self.H, self.W, self.T,
            self.dx, self.dy, self.dt, scale_log2, self.eps, self.tau_prime,
            cfg.bx, cfg.by, cfg.stride, cfg.radius,
            cfg.lam, cfg.theta, cfg.d_max, cfg.n_max,
            PREDICTORS.index(cfg.predictor))
        parts = [head]
        for sec in self.sections:
            payload = sec if cfg.backend == "identity" else zlib.compress(sec, 6)
            parts.append(struct.pack("<QQ", len(payload), len(sec)))
            parts.append(payload)
        return b"".join(parts)

    @classmethod
    def from_bytes(cls, blob: bytes) -> "Archive":
        """codec.py:255-282."""
        if len(blob) < _HEADER.size or blob[:4] != MAGIC:
            raise ValueError("not a VFCP archive")
        (magic, version, flags, H, W, T, dx, dy, dt, scale_log2, eps, tau,
         bx, by, stride, radius, lam, theta, d_max, n_max,
         pred_idx) = _HEADER.unpack_from(blob, 0)
        if version != VERSION:
            raise ValueError(f"unsupported archive version {version}")
        backend = "identity" if flags & FLAG_IDENTITY else "zlib"
        cfg = Config(predictor=PREDICTORS[pred_idx], bx=bx, by=by,
                     stride=stride, lam=lam, theta=theta, radius=radius,
                     d_max=d_max, n_max=n_max, backend=backend)
        off = _HEADER.size
        secs = []
        for _ in range(5):
            stored, raw = struct.unpack_from("<QQ", blob, off)
            off += 16
            payload = blob[off:off + stored]
            if len(payload) != stored:
                raise ValueError("truncated archive section")
            off += stored
            sec = payload if backend == "identity" else zlib.decompress(payload)
            if len(sec) != raw:
                raise ValueError("section length mismatch")
            secs.append(sec)
        return cls(H, W, T, dx, dy, dt, 2.0 ** scale_log2, eps, tau, cfg,
                   *secs)

    @property
    def nbytes(self) -> int:
        return len(self.to_bytes())

    def save(self, path) -> None:
        Path(path).write_bytes(self.to_bytes())

    @classmethod
    def load(cls, path) -> "Archive":
        return cls.from_bytes(Path(path).read_bytes())


@dataclass
class CompressStats:
    """codec.py:296-304."""
    symbols: np.ndarray
    signed_indices: np.ndarray
    overflow_count: int
    lossless_vertices: int
    modes: np.ndarray
    critical_faces: int


@dataclass(frozen=True)
class DecodeStats:
    """codec.py:307-314."""
    aux_component_buffers: int

    @property
    def aux_frames(self) -> float:
        return self.aux_component_buffers / 2.0


def _mode_grid_shape(H, W, cfg: Config):
    return (-(-H // cfg.by), -(-W // cfg.bx))


def make_params(H, W, T, dx, dy, dt, scale, tau, cfg: Config):
    p = _lib.vfcp_params()
    p.H, p.W, p.T = H, W, T
    p.dx, p.dy, p.dt = float(dx), float(dy), float(dt)
    p.scale = float(scale)
    p.tau = int(tau)
    p.predictor = _lib.PRED_INDEX[cfg.predictor]
    p.bx, p.by, p.stride = int(cfg.bx), int(cfg.by), int(cfg.stride)
    p.radius = int(cfg.radius)
    p.n_max = int(cfg.n_max)
    p.lam, p.theta, p.d_max = float(cfg.lam), float(cfg.theta), float(cfg.d_max)
    return p


def _sym_dtype(radius):
    import torch
    return torch.uint16 if radius <= 32768 else torch.int32


# --------------------------------------------------------------------------
# device pipeline (the hot path): field -> symbol streams

@dataclass
class DeviceStreams:
    """Device-resident outputs of the compress hot path (torch tensors)."""
    eps: float
    scale: float
    tau: int
    codes: object       # u8[N]
    ld: object          # u8[ceil(N/8)] np.packbits(xi == 0)
    qd: object          # u16 (or u32) symbols
    ll: object          # i64 lossless side stream
    modes: object       # u8[(T-1)*nby*nbx]
    mask: object = None  # u16[N] positive-face classes per anchor
    scores: object = None
    recon: object = None
    n_faces: int | None = None
    host: dict | None = None   # host copies (compress_device(host_out=True))
    hist: dict | None = None   # device symbol counts of qd / codes (want_hist)


def compress_device(f: FieldSeries, eps: float, config: Config | None = None,
                    relative: bool = False, want_mask: bool = False,
                    want_scores: bool = False, want_recon: bool = False,
                    host_out: bool = False,
                    want_hist: bool = False) -> DeviceStreams:
    """codec.py:321-376 up to (not including) the entropy stage, on device.

    host_out: also bring the streams to pinned host memory (``.host``),
    overlapping the copies with the encode: the codes and l_d right after
    the analysis, each frame's symbols as soon as the frame is encoded.
    want_hist: the frame-streamed path also counts the symbols of qd and the
    codes frame by frame (``.hist``, for the device entropy stage); the
    whole-field path leaves ``.hist`` None."""
    import torch
    cfg = config or Config()
    if eps < 0:
        raise ValueError("eps must be non-negative")
    H, W, T = f.H, f.W, f.T
    N = H * W * T
    L = _lib.lib()
    resident = None
    if _stream_ok(f, cfg, want_mask or want_scores or want_recon):
        # page-locked host input: frames are analysed and encoded while the
        # later ones are still crossing PCIe
        r = _compress_streamed(f, eps, cfg, relative, host_out, want_hist)
        if isinstance(r, DeviceStreams):
            return r
        resident = r    # left to the whole-field path below (already copied)
    du, dv = resident or (to_device(f.u), to_device(f.v))
    if du.dtype != dv.dtype:
        du, dv = du.double(), dv.double()
    lo, hi, ma = device_range(du, dv)
    if relative:
        eps = eps * (hi - lo)
    S = scale_for(ma)
    tau = tau_from_eps(eps, S)
    p = make_params(H, W, T, f.dx, f.dy, f.dt, S, tau, cfg)
    pp = ctypes.byref(p)
    st = _lib.stream_ptr()
    dev = du.device
    dt_code = dtype_code(du)
    codes = torch.empty(N, dtype=torch.uint8, device=dev)
    ld_words = torch.empty((N + 31) // 32, dtype=torch.int32, device=dev)
    mask = torch.empty(N, dtype=torch.int16, device=dev) if want_mask else None
    row_n31 = torch.empty(T * H, dtype=torch.int32, device=dev)
    _lib.check(L.vfcp_analyze(pp, du.data_ptr(), dv.data_ptr(), dt_code,
                              codes.data_ptr(), ld_words.data_ptr(),
                              _lib.ptr(mask), row_n31.data_ptr(), st),
               "analyze")
    qd_row_off = torch.empty(T * H + 1, dtype=torch.int64, device=dev)
    nqd = ctypes.c_int64(0)
    _lib.check(L.vfcp_qd_offsets(pp, row_n31.data_ptr(), qd_row_off.data_ptr(),
                                 ctypes.addressof(nqd), st), "qd offsets")
    nby, nbx = _mode_grid_shape(H, W, cfg)
    qd = torch.empty(max(nqd.value, 1), dtype=_sym_dtype(cfg.radius),
                     device=dev)
    modes = torch.empty(max((T - 1) * nby * nbx, 1), dtype=torch.uint8,
                        device=dev)
    scores = (torch.empty(max((T - 1) * nby * nbx * 2, 1), dtype=torch.float64,
                          device=dev) if want_scores else None)
    recon = (torch.empty(2 * N, dtype=torch.int64, device=dev)
             if want_recon else None)
    row_ll = torch.empty(T * H, dtype=torch.int32, device=dev)
    host = None
    if host_out and qd.dtype == torch.uint16 and not (want_scores or want_recon):
        # codes / l_d on a side stream while the encode runs
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(main)
        h_codes = torch.empty(N, dtype=torch.uint8, pin_memory=True)
        h_ld = torch.empty((N + 7) // 8, dtype=torch.uint8, pin_memory=True)
        with torch.cuda.stream(side):
            h_codes.copy_(codes, non_blocking=True)
            h_ld.copy_(ld_words.view(torch.uint8)[:(N + 7) // 8],
                       non_blocking=True)
        codes.record_stream(side)
        ld_words.record_stream(side)
        frame_off = qd_row_off[::H][:T + 1].cpu().numpy().astype(np.int64)
        h_qd = torch.empty(max(nqd.value, 1), dtype=torch.uint16,
                           pin_memory=True)
        _lib.check(L.vfcp_encode_host(
            pp, du.data_ptr(), dv.data_ptr(), dt_code, codes.data_ptr(),
            qd_row_off.data_ptr(), qd.data_ptr(), modes.data_ptr(),
            row_ll.data_ptr(), h_qd.data_ptr(), frame_off.ctypes.data, st),
            "encode (host out)")
        host = {"codes": h_codes, "ld": h_ld, "qd": h_qd[:nqd.value],
                "side": side}
    else:
        _lib.check(L.vfcp_encode(pp, du.data_ptr(), dv.data_ptr(), dt_code,
                                 codes.data_ptr(), qd_row_off.data_ptr(),
                                 qd.data_ptr(), modes.data_ptr(),
                                 _lib.ptr(scores), row_ll.data_ptr(),
                                 _lib.ptr(recon), st), "encode")
    return _finish_streams(f, cfg, p, du, dv, dt_code, eps, S, tau, codes,
                           ld_words, qd_row_off, nqd.value, qd, modes, row_ll,
                           mask, scores, recon, host)


def _finish_streams(f, cfg, p, du, dv, dt_code, eps, S, tau, codes, ld_words,
                    qd_row_off, nqd, qd, modes, row_ll, mask, scores, recon,
                    host):
    """The lossless side stream (codec.py:129-131,155-158), the host copies
    of the small streams, and the DeviceStreams record."""
    import torch
    L = _lib.lib()
    st = _lib.stream_ptr()
    pp = ctypes.byref(p)
    H, W, T = f.H, f.W, f.T
    N = H * W * T
    dev = du.device
    nby, nbx = _mode_grid_shape(H, W, cfg)
    ll_row_off = torch.empty(T * H + 1, dtype=torch.int64, device=dev)
    nll = ctypes.c_int64(0)
    _lib.check(L.vfcp_row_offsets(row_ll.data_ptr(), T * H,
                                  ll_row_off.data_ptr(), ctypes.addressof(nll),
                                  st), "ll offsets")
    ll = torch.empty(max(nll.value, 1), dtype=torch.int64, device=dev)
    if nll.value:
        _lib.check(L.vfcp_encode_ll(pp, du.data_ptr(), dv.data_ptr(), dt_code,
                                    codes.data_ptr(), qd.data_ptr(),
                                    qd_row_off.data_ptr(), row_ll.data_ptr(),
                                    ll_row_off.data_ptr(), ll.data_ptr(), st),
                   "encode ll")
    ld = ld_words.view(torch.uint8)[:(N + 7) // 8]
    if host is not None:
        side = host.pop("side")
        h_ll = _to_host(ll[:nll.value])
        h_modes = _to_host(modes[:(T - 1) * nby * nbx])
        torch.cuda.current_stream().synchronize()
        side.synchronize()
        host = {"codes": host["codes"].numpy(), "ld": host["ld"].numpy(),
                "qd": host["qd"].numpy(), "ll": h_ll.numpy(),
                "modes": h_modes.numpy()}
    return DeviceStreams(
        eps=eps, scale=S, tau=tau, codes=codes, ld=ld,
        qd=qd[:nqd], ll=ll[:nll.value],
        modes=modes[:(T - 1) * nby * nbx], mask=mask,
        scores=scores[:(T - 1) * nby * nbx * 2] if scores is not None else None,
        recon=recon, host=host)


# Below this many input bytes per frame the frame-streamed path's per-frame
# launches and host hand-shakes cost more than the overlap saves (configs 1-3:
# 0.1 - 2 MB frames, hundreds of frames; measured in
# profiles/bench_matrix_r02.json): such fields take the whole-field path.
STREAM_MIN_FRAME_BYTES = int(os.environ.get("VFCP_STREAM_MIN_FRAME_BYTES",
                                            str(16 << 20)))


def _stream_ok(f, cfg: Config, extras: bool) -> bool:
    """Whether compress_device may take the frame-streamed path: page-locked
    host tensors of one float dtype and a configuration of the block path
    (csrc/capi.cu fast_ok; tau' is checked once the range is known)."""
    if extras or os.environ.get("VFCP_NO_STREAM") or os.environ.get("VFCP_SLOW_PATH"):
        return False
    u, v = f.u, f.v
    if not (type(u).__module__.startswith("torch") and
            type(v).__module__.startswith("torch")):
        return False
    import torch
    if u.is_cuda or v.is_cuda or u.dtype != v.dtype:
        return False
    if u.dtype not in (torch.float32, torch.float64):
        return False
    if not (u.is_pinned() and v.is_pinned() and u.is_contiguous()
            and v.is_contiguous()):
        return False
    if 2 * f.H * f.W * u.element_size() < STREAM_MIN_FRAME_BYTES:
        return False
    return (cfg.bx == 32 and cfg.by == 32 and cfg.radius <= 32768
            and cfg.stride >= 2 and f.H <= 65535 and f.T >= 2)


def _compress_streamed(f: FieldSeries, eps: float, cfg: Config,
                       relative: bool, host_out: bool, want_hist: bool = False):
    """compress_device for a field in page-locked host memory, overlapped
    with its own H2D copy (codec.py:321-376; the result is the whole-field
    path's, stream for stream).

    The frames are copied one by one on a copy stream.  The scale S and a
    relative eps need the value range of the whole field before any vertex
    can be converted, so host threads reduce it at memory bandwidth while the
    first frames cross (vfcp_host_range); the device still reduces every
    frame as it arrives and the two must agree.  Frame t's codes are final
    once the anchors of frames t - 1 and t have been analysed
    (vfcp_analyze_slab), which needs frame t + 1 on the device; its symbol
    offsets follow from the counts of the frames before it; then the frame is
    encoded (vfcp_encode_stream_frame) and, with host_out, its codes / l_d /
    symbols go back on a side stream.  Returns the device copies (du, dv)
    instead when the configuration turns out to be outside the block path
    (tau', a list or int32 overflow): the caller then runs the whole-field
    path on them."""
    import torch
    L = _lib.lib()
    H, W, T = f.H, f.W, f.T
    HW = H * W
    N = HW * T
    hu, hv = f.u.reshape(-1), f.v.reshape(-1)
    dev = torch.device("cuda", torch.cuda.current_device())
    main = torch.cuda.current_stream()
    copy = torch.cuda.Stream()
    du = torch.empty(N, dtype=hu.dtype, device=dev)
    dv = torch.empty(N, dtype=hv.dtype, device=dev)
    dt_code = dtype_code(du)
    copy.wait_stream(main)
    arrived = []
    timing = bool(os.environ.get("VFCP_STREAM_TIMES"))
    if timing:
        import time
        w0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e0.record(copy)
    with torch.cuda.stream(copy):
        for t in range(T):
            a, b = t * HW, (t + 1) * HW
            du[a:b].copy_(hu[a:b], non_blocking=True)
            dv[a:b].copy_(hv[a:b], non_blocking=True)
            ev = torch.cuda.Event(enable_timing=timing)
            ev.record(copy)
            arrived.append(ev)
    du.record_stream(copy)
    dv.record_stream(copy)

    def whole_field():
        main.wait_stream(copy)
        return du, dv

    # The value range.  The device reduces every frame as it arrives (its own
    # stream, partial triples to page-locked memory); host threads reduce the
    # frames from the back of the field until they meet it: the frames the
    # DMA has not delivered yet are the ones only the host can see.
    # (More threads finish sooner but take memory bandwidth from the DMA; the
    # streams' D2H of host_out can only start once the range is known.)
    nthr = int(os.environ.get("VFCP_RANGE_THREADS", "0")) or \
        min(_lib.host_threads(), 16 if host_out else 8)
    nb = 8 * torch.cuda.get_device_properties(dev).multi_processor_count
    parts = torch.empty((T, nb, 3), dtype=torch.float64, device=dev)
    h_parts = torch.empty((T, nb, 3), dtype=torch.float64, pin_memory=True)
    esz = du.element_size()
    rstream = torch.cuda.Stream()
    rstream.wait_stream(main)
    rdone = []
    with torch.cuda.stream(rstream):
        for t in range(T):
            rstream.wait_event(arrived[t])
            _lib.check(L.vfcp_value_range_part(
                du.data_ptr() + t * HW * esz, dv.data_ptr() + t * HW * esz,
                dt_code, HW, parts[t].data_ptr(), nb, rstream.cuda_stream),
                "value_range part")
            h_parts[t].copy_(parts[t], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(rstream)
            rdone.append(ev)
    for x in (du, dv, parts):
        x.record_stream(rstream)
    hp = h_parts.numpy()
    out3 = np.zeros(3, np.float64)
    lo, hi, ma = math.inf, -math.inf, 0.0
    k = T
    while k > 0 and not rdone[k - 1].query():
        k -= 1
        _lib.check(L.vfcp_host_range(hu.data_ptr() + k * HW * esz,
                                     hv.data_ptr() + k * HW * esz, dt_code,
                                     HW, nthr, out3.ctypes.data), "host range")
        lo, hi, ma = min(lo, out3[0]), max(hi, out3[1]), max(ma, out3[2])
    host_frames = T - k
    if k > 0:
        rdone[k - 1].synchronize()
        lo = min(lo, hp[:k, :, 0].min())
        hi = max(hi, hp[:k, :, 1].max())
        ma = max(ma, hp[:k, :, 2].max())
    out3[:] = (lo, hi, ma)
    if timing:
        w1 = time.perf_counter()
    lo, hi, ma = float(out3[0]), float(out3[1]), float(out3[2])
    if relative:
        eps = eps * (hi - lo)
    S = scale_for(ma)
    tau = tau_from_eps(eps, S)
    if not 0 < tau < (1 << 29):
        return whole_field()
    p = make_params(H, W, T, f.dx, f.dy, f.dt, S, tau, cfg)
    pp = ctypes.byref(p)
    st = main.cuda_stream
    codes = torch.zeros(N, dtype=torch.uint8, device=dev)
    ld_words = torch.zeros((N + 31) // 32, dtype=torch.int32, device=dev)
    row_n31 = torch.zeros(T * H, dtype=torch.int32, device=dev)
    cap = min(HW, 1 << 25)
    lst = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    ovf = torch.zeros(1, dtype=torch.int32, device=dev)
    qd_row_off = torch.empty(T * H + 1, dtype=torch.int64, device=dev)
    qd = torch.empty(2 * N, dtype=torch.uint16, device=dev)
    nby, nbx = _mode_grid_shape(H, W, cfg)
    modes = torch.empty(max((T - 1) * nby * nbx, 1), dtype=torch.uint8,
                        device=dev)
    row_ll = torch.empty(T * H, dtype=torch.int32, device=dev)
    frame_off = torch.zeros(T + 1, dtype=torch.int64, pin_memory=True)
    fo = frame_off.numpy()
    side = h_codes = h_ld = h_qd = None
    ld_frames = HW % 32 == 0
    if host_out:
        side = torch.cuda.Stream()
        h_codes = torch.empty(N, dtype=torch.uint8, pin_memory=True)
        h_ld = torch.empty((N + 7) // 8, dtype=torch.uint8, pin_memory=True)
        h_qd = torch.empty(2 * N, dtype=torch.uint16, pin_memory=True)
    ld_bytes = ld_words.view(torch.uint8)
    hist = None
    if want_hist:
        hist = {"qd": torch.zeros(2 * cfg.radius, dtype=torch.int64, device=dev),
                "codes": torch.zeros(EB_ALPHABET, dtype=torch.int64, device=dev)}
        qd_base = max(0, cfg.radius - 4096)
    handle = ctypes.c_void_p()
    _lib.check(L.vfcp_encode_stream_begin(
        pp, du.data_ptr(), dv.data_ptr(), dt_code, codes.data_ptr(),
        qd_row_off.data_ptr(), qd.data_ptr(), modes.data_ptr(),
        row_ll.data_ptr(), st, ctypes.byref(handle)), "encode stream begin")
    try:
        main.wait_event(arrived[0])
        for t in range(T):
            if t + 1 < T:
                main.wait_event(arrived[t + 1])
            # the anchors of frame t (frames t, t + 1): frame t's codes final
            _lib.check(L.vfcp_analyze_slab(
                pp, du.data_ptr(), dv.data_ptr(), dt_code, t, t + 1,
                codes.data_ptr(), ld_words.data_ptr(), None,
                row_n31.data_ptr(), lst.data_ptr(), cap, count.data_ptr(),
                ovf.data_ptr(), st), "analyze slab")
            _lib.check(L.vfcp_qd_offsets_upto(
                pp, t + 1, row_n31.data_ptr(), qd_row_off.data_ptr(),
                frame_off.data_ptr() + 8 * (t + 1), st), "qd offsets")
            ready = torch.cuda.Event()
            ready.record(main)
            if host_out:
                side.wait_event(ready)
                with torch.cuda.stream(side):
                    a, b = t * HW, (t + 1) * HW
                    h_codes[a:b].copy_(codes[a:b], non_blocking=True)
                    if ld_frames:
                        h_ld[a // 8:b // 8].copy_(ld_bytes[a // 8:b // 8],
                                                  non_blocking=True)
            _lib.check(L.vfcp_encode_stream_frame(handle, t), "encode frame")
            if host_out:
                done = torch.cuda.Event()
                done.record(main)
            if host_out or want_hist:
                ready.synchronize()     # frame_off[t + 1] is on the host
                a, b = int(fo[t]), int(fo[t + 1])
            if host_out and b > a:
                side.wait_event(done)
                with torch.cuda.stream(side):
                    h_qd[a:b].copy_(qd[a:b], non_blocking=True)
            if want_hist:
                # symbol counts while the GPU waits for the next frame; the
                # spans are cut at multiples of 8 symbols (16-byte loads)
                a8 = a & ~7
                b8 = b if t == T - 1 else b & ~7
                _lib.check(L.vfcp_huff_hist_dev(
                    qd.data_ptr() + 2 * a8, 2, b8 - a8, 2 * cfg.radius, qd_base,
                    hist["qd"].data_ptr(), st), "huffman histogram")
                _lib.check(L.vfcp_huff_hist_dev(
                    codes.data_ptr() + t * HW, 1, HW, EB_ALPHABET, 0,
                    hist["codes"].data_ptr(), st), "huffman histogram")
    except BaseException:
        L.vfcp_encode_stream_end(handle, None)
        raise
    h_ovf = torch.empty(1, dtype=torch.int32, pin_memory=True)
    h_ovf.copy_(ovf, non_blocking=True)
    enc_ovf = ctypes.c_int(0)
    _lib.check(L.vfcp_encode_stream_end(handle, ctypes.byref(enc_ovf)),
               "encode stream end")      # synchronises the main stream
    if timing:
        w2 = time.perf_counter()
        import sys
        print(f"[stream] range known after {1e3 * (w1 - w0):.1f} ms ({nthr} "
              f"threads took the last {host_frames} frames); "
              f"frames on device at "
              + " ".join(f"{e0.elapsed_time(a):.0f}" for a in arrived)
              + f" ms; main stream done {1e3 * (w2 - w0):.1f} ms",
              file=sys.stderr)
    # the device's own range of every frame against the one used above
    rdone[T - 1].synchronize()
    c = (float(hp[:, :, 0].min()), float(hp[:, :, 1].max()),
         float(hp[:, :, 2].max()))
    if c != (lo, hi, ma):
        raise _lib.VfcpError(
            f"host and device value ranges disagree: {(lo, hi, ma)} vs {c}")
    if enc_ovf.value or int(h_ovf[0]) != 0:
        if side is not None:
            side.synchronize()
        return whole_field()
    nqd = int(fo[T])
    host = None
    if host_out:
        if not ld_frames:
            side.wait_stream(main)
            with torch.cuda.stream(side):
                h_ld.copy_(ld_bytes[:(N + 7) // 8], non_blocking=True)
        for x in (codes, ld_words, qd):
            x.record_stream(side)
        host = {"codes": h_codes, "ld": h_ld, "qd": h_qd[:nqd], "side": side}
    s = _finish_streams(f, cfg, p, du, dv, dt_code, eps, S, tau, codes,
                        ld_words, qd_row_off, nqd, qd, modes, row_ll,
                        None, None, None, host)
    s.hist = hist
    return s


def archive_from_streams(f_dims, s: DeviceStreams, cfg: Config,
                         host=None) -> Archive:
    """Host entropy stage (codec.py:378-387): Huffman + packbits."""
    H, W, T, dx, dy, dt = f_dims
    h = host or streams_to_host(s)
    nby, nbx = _mode_grid_shape(H, W, cfg)
    return Archive(
        H=H, W=W, T=T, dx=dx, dy=dy, dt=dt, scale=s.scale, eps=s.eps,
        tau_prime=s.tau, config=cfg,
        q_xi=huffman.encode(h["codes"], EB_ALPHABET),
        q_d=huffman.encode(h["qd"], 2 * cfg.radius),
        l_d=h["ld"].tobytes(),
        lossless_stream=h["ll"].astype("<i8").tobytes(),
        mode_bitmap=np.packbits(h["modes"]).tobytes(),
    )


def _to_host(x):
    """D2H into pinned memory (torch's caching host allocator reuses it):
    pageable copies of gigabyte streams are several times slower."""
    import torch
    h = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
    h.copy_(x, non_blocking=True)
    return h


def streams_to_host(s: DeviceStreams) -> dict:
    import torch
    if s.host is not None:
        return s.host
    hs = {k: _to_host(getattr(s, k)) for k in ("codes", "ld", "qd", "ll", "modes")}
    torch.cuda.current_stream().synchronize()
    return {k: v.numpy() for k, v in hs.items()}


def compress(f: FieldSeries, eps: float, config: Config | None = None,
             relative: bool = False) -> Archive:
    """Compress a field series under a uniform pointwise error bound eps.

    codec.py:321-398.  With relative=True, eps is a fraction of the joint
    value range.  Every critical-point trajectory of the input is preserved
    exactly by construction."""
    cfg = config or Config()
    if not cfg.stats and cfg.radius <= 32768:
        # entropy stage on the device (csrc/huffman_gpu.cu): only the packed
        # sections come back; zlib stays on the host
        import torch
        # (the codes' section is built after the frames: its kernels, run
        # beside the frame loop on a side stream, take issue slots from the
        # block-scan chain and the call ends later)
        timing = bool(os.environ.get("VFCP_ARCHIVE_TIMES"))
        if timing:
            import time
            tm = [time.perf_counter()]
            mark = lambda: tm.append(time.perf_counter())   # noqa: E731
        else:
            mark = lambda: None   # noqa: E731
        s = compress_device(f, eps, cfg, relative, want_hist=True)
        mark()
        hq, hc = (s.hist["qd"], s.hist["codes"]) if s.hist else (None, None)
        # the small sections go to pinned memory on a side stream while
        # the symbol section is histogrammed and packed
        main = torch.cuda.current_stream()
        side = torch.cuda.Stream()
        side.wait_stream(main)
        with torch.cuda.stream(side):
            h_ld, h_ll, h_modes = _to_host(s.ld), _to_host(s.ll), _to_host(s.modes)
        for x in (s.ld, s.ll, s.modes):
            x.record_stream(side)
        pending = huffman.encode_device_many([
            (s.qd, 2 * cfg.radius, max(0, cfg.radius - 4096), hq),
            (s.codes, EB_ALPHABET, 0, hc)])
        mark()
        side.synchronize()
        l_d = memoryview(h_ld.numpy())     # page-locked, no second copy
        mark()
        q_d = pending[0].result()
        q_xi = pending[1].result()
        mark()
        a = Archive(
            H=f.H, W=f.W, T=f.T, dx=f.dx, dy=f.dy, dt=f.dt, scale=s.scale,
            eps=s.eps, tau_prime=s.tau, config=cfg, q_xi=q_xi, q_d=q_d,
            l_d=l_d,
            lossless_stream=h_ll.numpy().astype("<i8", copy=False).tobytes(),
            mode_bitmap=np.packbits(h_modes.numpy()).tobytes(),
        )
        if timing:
            mark()
            import sys
            d = [1e3 * (tm[i + 1] - tm[i]) for i in range(len(tm) - 1)]
            print(f"[archive] compress_device {d[0]:.1f} | small D2H + pack "
                  f"enqueue {d[1]:.1f} | l_d bytes {d[2]:.1f} | q_d, q_xi "
                  f"bytes {d[3]:.1f} | Archive {d[4]:.1f} ms", file=sys.stderr)
        return a
    s = compress_device(f, eps, cfg, relative, want_mask=cfg.stats,
                        host_out=True)
    host = streams_to_host(s)
    a = archive_from_streams((f.H, f.W, f.T, f.dx, f.dy, f.dt), s, cfg, host)
    if cfg.stats:
        qd = host["qd"].astype(np.int32)
        nby, nbx = _mode_grid_shape(f.H, f.W, cfg)
        mask = s.mask.cpu().numpy().view(np.uint16)
        n_faces = int(np.unpackbits(mask.view(np.uint8)).sum())
        a.stats = CompressStats(
            symbols=qd.copy(),
            signed_indices=(qd[qd != 0] - cfg.radius).astype(np.int32),
            overflow_count=int((qd == 0).sum()),
            lossless_vertices=int(np.unpackbits(host["ld"])[:f.n_samples].sum()),
            modes=host["modes"].reshape(max(f.T - 1, 0), nby, nbx),
            critical_faces=n_faces,
        )
    return a


# --------------------------------------------------------------------------
# decompression

class _SideDecode:
    """huffman.decode_device on a host thread and a side stream."""

    def __init__(self, blob, dtype):
        import threading

        import torch
        self._out = self._err = None
        dev = torch.cuda.current_device()

        def work():
            try:
                with torch.cuda.device(dev):
                    side = torch.cuda.Stream()
                    with torch.cuda.stream(side):
                        self._out = huffman.decode_device(blob, dtype)
                    side.synchronize()
            except BaseException as err:
                self._err = err

        self._t = threading.Thread(target=work, daemon=True)
        self._t.start()

    def result(self):
        import torch
        self._t.join()
        if self._err is not None:
            raise self._err
        if self._out.numel():
            self._out.record_stream(torch.cuda.current_stream())
        return self._out


def _clamp_codes(blob):
    """Codes of a q_xi section whose alphabet exceeds 32, mapped to the
    code with the same ladder step (codec.py:427-431 eq = tau >> min(code,
    K_MAX), 0 for code 31): 31 stays 31, anything else above K_MAX becomes
    K_MAX.  Decoded wide (uint16 on the device, or int64 on the host for an
    alphabet past 2^16), so no code aliases to 31 by truncation."""
    import torch
    if huffman.alphabet_of(blob) <= 65536:
        c = huffman.decode_device(blob, np.uint16).to(torch.int32)
    else:
        c = torch.from_numpy(huffman.decode(blob, np.int64)).cuda()
    c = torch.where(c == CODE_LOSSLESS, c, c.clamp(max=K_MAX))
    return c.to(torch.uint8)


def decompress_device(a: Archive, want_fixed: bool = False, codes=None,
                      qd=None, ll=None, modes=None, ld=None, host_out=None):
    """codec.py:401-453 on device.  Returns (out_u, out_v, fix_u, fix_v)
    as CUDA tensors.  codes/qd/ll/modes may be passed pre-decoded (host
    numpy or device tensors) to skip the host entropy stage.  host_out:
    (u, v) page-locked float64 host tensors that receive each frame's output
    while later frames decode (not with want_fixed)."""
    import torch
    cfg = a.config
    n = a.H * a.W * a.T
    qd_pre = qd_err = None
    if codes is None:
        # entropy decode on the device (huffman.decode_device); with the
        # symbol section also to decode, the codes go to a host thread on a
        # side stream and both sections decode concurrently (errors are
        # raised in the sequential order: codes first)
        if huffman.alphabet_of(a.q_xi) > EB_ALPHABET:
            # a q_xi section with codes >= 32 (never written by compress):
            # the reference reads them through tau >> min(code, K_MAX), so
            # every code other than 31 above K_MAX acts as K_MAX
            codes = _clamp_codes(a.q_xi)
        elif qd is None and cfg.radius <= 32768:
            th = _SideDecode(a.q_xi, np.uint8)
            try:
                qd_pre = huffman.decode_device(a.q_d, np.uint16)
            except ValueError as err:
                qd_err = err
            codes = th.result()
        else:
            codes = huffman.decode_device(a.q_xi, np.uint8)
    if codes.shape[0] != n:
        raise ValueError("eb code stream length mismatch")
    if len(a.l_d) < (n + 7) // 8:
        # np.unpackbits(...)[:n] is shorter than n: never equal to eq == 0
        raise ValueError("lossless bitmap disagrees with eb codes")
    if qd is None:
        if cfg.radius <= 32768:
            if qd_err is not None:
                raise qd_err
            qd = (qd_pre if qd_pre is not None
                  else huffman.decode_device(a.q_d, np.uint16))
            # any symbol >= 2 radius (uint16 seen as int16: no uint16 max)
            q16, lim = qd.view(torch.int16), 2 * cfg.radius
            if lim >= 65536:
                bad = False
            elif lim <= 32768:
                bad = bool(((q16 < 0) | (q16 >= lim)).any().item())
            else:
                bad = bool(((q16 < 0) & (q16 >= lim - 65536)).any().item())
        else:
            qd = huffman.decode(a.q_d, np.uint32)
            bad = qd.size and int(qd.max()) >= 2 * cfg.radius
        if bad:
            raise ValueError("corrupt entropy stream")
    if ll is None:
        ll = np.frombuffer(a.lossless_stream, dtype="<i8").astype(np.int64)
    nby, nbx = _mode_grid_shape(a.H, a.W, cfg)
    if modes is None:
        n_mode_bits = max(a.T - 1, 0) * nby * nbx
        mode_bits = np.unpackbits(
            np.frombuffer(a.mode_bitmap, dtype=np.uint8))[:n_mode_bits]
        modes = mode_bits.reshape(max(a.T - 1, 0), nby, nbx).astype(
            np.uint8).reshape(-1)

    def dev(x, dt=None):
        if type(x).__module__.startswith("torch"):
            return x.cuda().contiguous()
        x = np.ascontiguousarray(x)
        if not x.flags.writeable:
            x = x.copy()
        return torch.from_numpy(x).cuda()

    d_codes = dev(codes)
    d_ld = dev(ld if ld is not None else
               np.frombuffer(a.l_d, dtype=np.uint8)[:(n + 7) // 8])
    d_qd = dev(qd)
    if d_qd.dtype == torch.int32 and cfg.radius <= 32768:
        d_qd = d_qd.to(torch.uint16)
    d_ll = dev(ll) if len(ll) else torch.zeros(1, dtype=torch.int64,
                                                device="cuda")
    d_modes = dev(modes) if len(modes) else torch.zeros(1, dtype=torch.uint8,
                                                        device="cuda")
    p = make_params(a.H, a.W, a.T, a.dx, a.dy, a.dt, a.scale, a.tau_prime, cfg)
    pp = ctypes.byref(p)
    L = _lib.lib()
    st = _lib.stream_ptr()
    nrows = a.T * a.H
    row_n31 = torch.empty(nrows, dtype=torch.int32, device="cuda")
    row_ll = torch.empty(nrows, dtype=torch.int32, device="cuda")
    qd_row_off = torch.empty(nrows + 1, dtype=torch.int64, device="cuda")
    ll_row_off = torch.empty(nrows + 1, dtype=torch.int64, device="cuda")
    totals = np.zeros(2, np.int64)
    ld_ok = ctypes.c_int(1)
    n_qd = int(d_qd.numel()) if len(qd) else 0
    if n_qd == 0:
        d_qd = torch.zeros(1, dtype=d_qd.dtype, device="cuda")
    _lib.check(L.vfcp_decode_prepare(
        pp, d_codes.data_ptr(), d_ld.data_ptr(), d_qd.data_ptr(), n_qd,
        row_n31.data_ptr(), qd_row_off.data_ptr(), row_ll.data_ptr(),
        ll_row_off.data_ptr(), totals.ctypes.data, ctypes.addressof(ld_ok),
        st), "decode prepare")
    if not ld_ok.value:
        raise ValueError("lossless bitmap disagrees with eb codes")
    if totals[0] != n_qd:
        raise ValueError("residual stream length mismatch")
    if totals[1] != len(ll):
        raise ValueError("lossless stream length mismatch")
    out_u = torch.empty(n, dtype=torch.float64, device="cuda")
    out_v = torch.empty(n, dtype=torch.float64, device="cuda")
    fix_u = torch.empty(n, dtype=torch.int64, device="cuda") if want_fixed else None
    fix_v = torch.empty(n, dtype=torch.int64, device="cuda") if want_fixed else None
    if host_out is not None and not want_fixed:
        hu, hv = host_out
        if hu.numel() != n or hv.numel() != n or hu.dtype != torch.float64:
            raise ValueError("host_out: two float64 host tensors of H*W*T")
        _lib.check(L.vfcp_decode_host(pp, d_codes.data_ptr(), d_qd.data_ptr(),
                                      n_qd, d_ll.data_ptr(), len(ll),
                                      d_modes.data_ptr(), qd_row_off.data_ptr(),
                                      ll_row_off.data_ptr(), out_u.data_ptr(),
                                      out_v.data_ptr(), hu.data_ptr(),
                                      hv.data_ptr(), st), "decode")
    else:
        _lib.check(L.vfcp_decode(pp, d_codes.data_ptr(), d_qd.data_ptr(), n_qd,
                                 d_ll.data_ptr(), len(ll), d_modes.data_ptr(),
                                 qd_row_off.data_ptr(), ll_row_off.data_ptr(),
                                 out_u.data_ptr(), out_v.data_ptr(),
                                 _lib.ptr(fix_u), _lib.ptr(fix_v), st), "decode")
    return out_u, out_v, fix_u, fix_v


def decompress_with_stats(a: Archive) -> tuple[FieldSeries, DecodeStats]:
    import torch
    n = a.H * a.W * a.T
    # each frame's output comes back to pinned memory while later frames
    # decode; FieldSeries re-validates the output (codec.py:451) on the
    # device
    hu = torch.empty(n, dtype=torch.float64, pin_memory=True)
    hv = torch.empty(n, dtype=torch.float64, pin_memory=True)
    out_u, out_v, _, _ = decompress_device(a, host_out=(hu, hv))
    fs = FieldSeries(a.H, a.W, a.T, a.dx, a.dy, a.dt, out_u, out_v)
    torch.cuda.current_stream().synchronize()
    object.__setattr__(fs, "u", hu.numpy())
    object.__setattr__(fs, "v", hv.numpy())
    return fs, DecodeStats(aux_component_buffers=4)


def decompress(a: Archive) -> FieldSeries:
    return decompress_with_stats(a)[0]


def reconstruct_fixed(a: Archive) -> FixedField:
    """Reconstruction as integers at the archive's scale (codec.py:460-463)."""
    import torch
    _, _, fu, fv = decompress_device(a, want_fixed=True)
    hu, hv = _to_host(fu), _to_host(fv)
    torch.cuda.current_stream().synchronize()
    return FixedField(a.H, a.W, a.T, hu.numpy(), hv.numpy(), a.scale)
