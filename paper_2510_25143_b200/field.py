"""Field data model and the fixed-point bridge (field.py of the reference).

FieldSeries / FixedField mirror the reference dataclasses (field.py:26-91):
same fields, same validation, same errors.  Components may be numpy arrays
(the reference's contract) or torch CUDA tensors already resident in HBM
(used by the benchmark); everything downstream accepts both.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib

FIXED_LIMIT = 1 << 30


class FieldError(ValueError):
    pass


def _is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


@dataclass(frozen=True)
class FieldSeries:
    H: int
    W: int
    T: int
    dx: float
    dy: float
    dt: float
    u: object  # float array of length H*W*T (numpy, or a torch CUDA tensor)
    v: object

    def __post_init__(self):
        # field.py:37-51
        if self.H < 2 or self.W < 2 or self.T < 2:
            raise FieldError(f"dims must be >= 2, got {self.H}x{self.W}x{self.T}")
        if self.dx <= 0 or self.dy <= 0 or self.dt <= 0:
            raise FieldError("dx, dy, dt must be positive")
        n = self.H * self.W * self.T
        if tuple(self.u.shape) != (n,) or tuple(self.v.shape) != (n,):
            raise FieldError(
                f"component length mismatch: expected {n}, "
                f"got u={tuple(self.u.shape)} v={tuple(self.v.shape)}")
        for name, arr in (("u", self.u), ("v", self.v)):
            if _is_torch(arr):
                import torch
                # (one reduction; the index list only for a field that fails)
                if not bool(torch.isfinite(arr).all()):
                    bad = torch.nonzero(~torch.isfinite(arr))
                    raise FieldError(
                        f"non-finite sample in {name} at index {int(bad[0, 0])}")
            else:
                bad = np.flatnonzero(~np.isfinite(arr))
                if bad.size:
                    raise FieldError(
                        f"non-finite sample in {name} at index {int(bad[0])}")

    @property
    def n_samples(self) -> int:
        return self.H * self.W * self.T

    @property
    def nbytes(self) -> int:
        """Raw size of the original data (both components, float32)."""
        return self.n_samples * 2 * 4

    def vid(self, t: int, i: int, j: int) -> int:
        return t * self.H * self.W + i * self.W + j

    def frames(self, comp: str):
        arr = self.u if comp == "u" else self.v
        return arr.reshape(self.T, self.H, self.W)

    def value_range(self) -> float:
        """Joint (u, v) max - min (field.py:69-73), reduced on the device."""
        lo, hi, _ = device_range(self.u, self.v)
        return hi - lo


@dataclass(frozen=True)
class FixedField:
    H: int
    W: int
    T: int
    u_fp: object  # int64 fixed values, length H*W*T
    v_fp: object
    scale: float

    @property
    def n_samples(self) -> int:
        return self.H * self.W * self.T

    def frames(self, comp: str):
        arr = self.u_fp if comp == "u" else self.v_fp
        return arr.reshape(self.T, self.H, self.W)


@dataclass(frozen=True)
class QualityReport:
    psnr_u: float
    psnr_v: float
    psnr_joint: float
    max_abs_err: float
    cr: float


# ---------------------------------------------------------------- device I/O

def to_device(a):
    """Float component -> contiguous CUDA tensor (float32 or float64)."""
    import torch
    if _is_torch(a):
        t = a
        if t.dtype not in (torch.float32, torch.float64):
            t = t.to(torch.float64)
        if not t.is_cuda:
            t = t.cuda(non_blocking=True)
        return t.contiguous()
    arr = np.ascontiguousarray(a)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)
    return torch.from_numpy(arr).cuda()


def dtype_code(t) -> int:
    import torch
    return _lib.VFCP_F32 if t.dtype == torch.float32 else _lib.VFCP_F64


def device_range(u, v):
    """(min, max, max|x|) over both components, exact (K0)."""
    du, dv = to_device(u), to_device(v)
    if du.dtype != dv.dtype:
        du, dv = du.double(), dv.double()
    out = np.zeros(3, np.float64)
    _lib.check(_lib.lib().vfcp_value_range(
        du.data_ptr(), dv.data_ptr(), dtype_code(du), du.numel(),
        out.ctypes.data, _lib.stream_ptr()), "value_range")
    return float(out[0]), float(out[1]), float(out[2])


# ---------------------------------------------------------- fixed-point bridge

def round_half_away(x):
    """Round half away from zero, elementwise, to int64 (field.py:295-297)."""
    return (np.sign(x) * np.floor(np.abs(x) + 0.5)).astype(np.int64)


def choose_scale(max_abs: float) -> float:
    """Largest power of two S with max_abs*S < 2^30 (field.py:300-310)."""
    if max_abs == 0.0:
        return float(FIXED_LIMIT)
    k = int(math.floor(math.log2(FIXED_LIMIT / max_abs)))
    s = 2.0 ** k
    while max_abs * s >= FIXED_LIMIT:
        s /= 2.0
    while max_abs * (s * 2.0) < FIXED_LIMIT:
        s *= 2.0
    return s


def scale_for(max_abs: float) -> float:
    """to_fixed's automatic scale including its retry loop (field.py:323-331).

    x -> rha(x*S) is monotone in |x|, so the largest fixed magnitude is
    rha(max_abs*S) and the retry test needs no pass over the data."""
    s = choose_scale(max_abs)
    while math.floor(max_abs * s + 0.5) >= FIXED_LIMIT:
        s /= 2.0
    return s


def to_fixed(f: FieldSeries, scale: float | None = None) -> FixedField:
    """S-scaled int64 fixed values (field.py:313-336), converted on device."""
    import torch
    du, dv = to_device(f.u), to_device(f.v)
    if scale is None:
        _, _, ma = device_range(du, dv)
        s = scale_for(ma)
    else:
        s = float(scale)
    # the conversion is elementwise IEEE float64; torch's CUDA ops are exact
    # for x*S (power of two), abs, +0.5 and floor
    def conv(t):
        y = t.double() * s
        return (torch.sign(y) * torch.floor(torch.abs(y) + 0.5)).to(torch.int64)
    return FixedField(f.H, f.W, f.T, conv(du).cpu().numpy(),
                      conv(dv).cpu().numpy(), s)


def from_fixed(ff: FixedField, dx=1.0, dy=1.0, dt=1.0) -> FieldSeries:
    """Exact float64 image of the fixed values (field.py:339-343)."""
    return FieldSeries(ff.H, ff.W, ff.T, dx, dy, dt,
                       np.asarray(ff.u_fp) / ff.scale,
                       np.asarray(ff.v_fp) / ff.scale)


def psnr(orig: FieldSeries, recon: FieldSeries, archive_size: int | None = None
         ) -> QualityReport:
    """field.py:346-372 (host, reporting only)."""
    if (orig.H, orig.W, orig.T) != (recon.H, recon.W, recon.T):
        raise FieldError("dimension mismatch between original and reconstruction")
    ou = np.asarray(_host(orig.u), np.float64)
    ov = np.asarray(_host(orig.v), np.float64)
    ru = np.asarray(_host(recon.u), np.float64)
    rv = np.asarray(_host(recon.v), np.float64)
    lo = min(float(ou.min()), float(ov.min()))
    hi = max(float(ou.max()), float(ov.max()))
    rng = hi - lo
    du = ou - ru
    dv = ov - rv

    def _psnr(mse):
        if mse == 0.0:
            return math.inf
        if rng == 0.0:
            return -math.inf
        return 20.0 * math.log10(rng) - 10.0 * math.log10(mse)

    mse_u = float(np.mean(du * du))
    mse_v = float(np.mean(dv * dv))
    max_err = max(float(np.abs(du).max()), float(np.abs(dv).max()))
    cr = orig.nbytes / archive_size if archive_size else float("nan")
    return QualityReport(psnr_u=_psnr(mse_u), psnr_v=_psnr(mse_v),
                         psnr_joint=_psnr(0.5 * (mse_u + mse_v)),
                         max_abs_err=max_err, cr=cr)


def _host(a):
    if _is_torch(a):
        return a.detach().cpu().numpy()
    return a


# ------------------------------------------------------------- raw I/O
# field.py:103-138: headerless little-endian float32 components plus a JSON
# sidecar with the dims and spacing.  Components are read straight into
# page-locked host memory, so compress() moves them to the GPU at PCIe rate.

def _pinned_f32(n: int) -> np.ndarray:
    try:
        import torch
        if torch.cuda.is_available():
            return torch.empty(n, dtype=torch.float32, pin_memory=True).numpy()
    except Exception:   # pragma: no cover - no torch / no driver
        pass
    return np.empty(n, dtype=np.float32)


def load_raw(u_path, v_path, H, W, T, dx=1.0, dy=1.0, dt=1.0) -> FieldSeries:
    """Two headerless little-endian float32 binaries of H*W*T samples each
    (field.py:103-116: the same size check and message)."""
    from pathlib import Path
    n = H * W * T
    comps = {}
    for name, path in (("u", u_path), ("v", v_path)):
        path = Path(path)
        actual = path.stat().st_size
        expected = n * 4
        if actual != expected:
            raise FieldError(
                f"{path}: expected {expected} bytes ({n} float32), got {actual}")
        a = _pinned_f32(n)
        with path.open("rb") as fh:
            got = fh.readinto(memoryview(a).cast("B"))
        if got != expected:   # pragma: no cover - file shrank under us
            raise FieldError(f"{path}: short read ({got} of {expected} bytes)")
        if np.little_endian is False:   # pragma: no cover
            a.byteswap(inplace=True)
        comps[name] = a
    return FieldSeries(H, W, T, dx, dy, dt, comps["u"], comps["v"])


def save_raw(f: FieldSeries, u_path, v_path, meta_path=None) -> None:
    """field.py:119-124."""
    import json
    from pathlib import Path
    np.asarray(_host(f.u)).astype("<f4").tofile(u_path)
    np.asarray(_host(f.v)).astype("<f4").tofile(v_path)
    if meta_path is not None:
        meta = {"H": f.H, "W": f.W, "T": f.T, "dx": f.dx, "dy": f.dy, "dt": f.dt}
        Path(meta_path).write_text(json.dumps(meta, indent=2) + "\n")


def load_meta(meta_path) -> dict:
    """field.py:127-136."""
    import json
    from pathlib import Path
    meta = json.loads(Path(meta_path).read_text())
    for key in ("H", "W", "T"):
        if key not in meta:
            raise FieldError(f"metadata sidecar missing '{key}'")
    meta.setdefault("dx", 1.0)
    meta.setdefault("dy", 1.0)
    meta.setdefault("dt", 1.0)
    return meta
