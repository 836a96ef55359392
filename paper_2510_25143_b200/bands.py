"""Row-band sharding of the analysis stage (first step).

The compress path's first two stages shard by row bands with no data-path
exchange beyond one halo row:

* range / scale (codec.py:332-333, field.py:313-336): every rank reduces
  its own band on the device (`vfcp_value_range`), then one MIN all-reduce
  of (min, -max, -max|x|) gives every rank the global range, the relative
  eps and the fixed-point scale S (min and max are exact element values,
  so the result does not depend on the split);
* analysis (faces, SoS, edge bounds, codes, `l_d`; predicates.py:270-301,
  ebounds.py:101-206, codec.py:71-115): a vertex's bound is a min over the
  faces that contain it, and those are anchored in its own row and the row
  above and span at most the row below, so band rows [r0, r1) analysed as
  the sub-field of rows [r0 - 1, r1 + 1) (clamped) at the global S and tau'
  give exactly the global codes for those rows.  The SoS tie-break ranks
  vertices by id only through comparisons, and the sub-field's ids keep the
  global order, so degenerate faces resolve the same way.

The encode that follows needs, per frame, the reconstructed last row of the
band above (Lorenzo) and R rows of the previous frame's reconstruction
(semi-Lagrangian); that exchange is not built, so bench.py
still runs replicas.  Backend-agnostic: NCCL on the GPU box, gloo in the
CPU tests (tests/test_multiproc.py).
"""

from __future__ import annotations

import ctypes

from . import _lib
from .field import dtype_code, scale_for, to_device


def band_rows(H: int, rank: int, world: int):
    """Rows [r0, r1) of band `rank`: contiguous, balanced to within a row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    q, r = divmod(H, world)
    r0 = rank * q + min(rank, r)
    return r0, r0 + q + (1 if rank < r else 0)


def halo_rows(H: int, r0: int, r1: int):
    """Rows [h0, h1) to analyse for band [r0, r1): one halo row each side."""
    return max(0, r0 - 1), min(H, r1 + 1)


def reduce_range(lo: float, hi: float, ma: float, dist=None, device="cuda"):
    """Global (min, max, max|x|) from per-band values: one all-reduce."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return lo, hi, ma
    import torch
    t = torch.tensor([lo, -hi, -ma], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    return float(t[0]), -float(t[1]), -float(t[2])


def band_scale(lo, hi, ma, eps, relative, dist=None, device="cuda"):
    """(eps_abs, S) for the whole field from a band's own range."""
    lo, hi, ma = reduce_range(lo, hi, ma, dist, device)
    if relative:
        eps = eps * (hi - lo)
    return eps, scale_for(ma)


def analyze_band(u_band, v_band, H: int, W: int, T: int, r0: int, r1: int,
                 scale: float, tau: int, cfg=None):
    """Codes u8[T, r1 - r0, W] of band rows [r0, r1), from the band's
    sub-field with its halo rows: `u_band`/`v_band` hold rows [h0, h1) of
    every frame (halo_rows), frame-major, on the device."""
    import torch
    from .codec import Config, make_params
    h0, h1 = halo_rows(H, r0, r1)
    Hb = h1 - h0
    du, dv = to_device(u_band), to_device(v_band)
    if du.numel() != Hb * W * T or dv.numel() != du.numel():
        raise ValueError("band arrays must hold rows [h0, h1) of every frame")
    N = Hb * W * T
    p = make_params(Hb, W, T, 1.0, 1.0, 1.0, scale, tau, cfg or Config())
    codes = torch.empty(N, dtype=torch.uint8, device=du.device)
    ld = torch.empty((N + 31) // 32, dtype=torch.int32, device=du.device)
    row = torch.empty(T * Hb, dtype=torch.int32, device=du.device)
    _lib.check(_lib.lib().vfcp_analyze(
        ctypes.byref(p), du.data_ptr(), dv.data_ptr(), dtype_code(du),
        codes.data_ptr(), ld.data_ptr(), _lib.ptr(None), row.data_ptr(),
        _lib.stream_ptr()), "analyze (band)")
    return codes.view(T, Hb, W)[:, r0 - h0:r1 - h0]


def face_mask_band(u_band, v_band, H: int, W: int, T: int, r0: int, r1: int,
                   scale: float):
    """12-bit positive-face mask i16[T, r1 - r0, W] of the faces anchored in
    band rows [r0, r1) (the K7 mask of `verify`, tracking.py:170-195).
    `u_band`/`v_band` hold the band with its halo rows, rows [h0, h1) of
    every frame (halo_rows, as analyze_band): a face spans its anchor row and
    the row below, and the row above keeps the sub-field at least two rows
    tall for one-row bands (its anchors are dropped; SoS compares vertex ids
    only by order, which the sub-field keeps).  An empty band (more ranks
    than rows) gives an empty mask.  Per-band flipped-face counts add up
    across ranks (one SUM all-reduce of fc_t, fc_s)."""
    import torch

    from .predicates import face_mask_float
    h0, h1 = halo_rows(H, r0, r1)
    Hb = max(0, h1 - h0)
    du, dv = to_device(u_band), to_device(v_band)
    if du.numel() != Hb * W * T or dv.numel() != du.numel():
        raise ValueError("band arrays must hold rows [h0, h1) of every frame")
    if r1 <= r0:
        return torch.zeros((T, 0, W), dtype=torch.int16, device=du.device)
    m = face_mask_float(Hb, W, T, du, dv, scale, host=False)
    return m.view(T, Hb, W)[:, r0 - h0:r1 - h0]


def flipped_faces(mask_a, mask_b):
    """(fc_t, fc_s) between two masks of the same faces (slice classes are
    bits 0-1, slab classes bits 2-11), counted on the device."""
    import torch

    from .tracking import _popcount12
    x = (mask_a.to(torch.int32) ^ mask_b.to(torch.int32)) & 0xFFF
    return _popcount12(x & 0x3), _popcount12(x & 0xFFC)


def sum_counts(counts, dist=None, device="cuda"):
    """Whole-field (fc_t, fc_s) from per-band counts: one SUM all-reduce."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return tuple(int(c) for c in counts)
    import torch
    t = torch.tensor(list(counts), dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return tuple(int(c) for c in t.tolist())
