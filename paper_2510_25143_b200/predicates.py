"""Critical-face set on the device (predicates.py:138-150, 290-301).

The analysis kernel (csrc/analyze.cu) evaluates the exact SoS face predicate
for every face of the implicit space-time mesh and returns a 12-bit class
mask per anchor vertex; this module converts it to the reference's
CriticalFaceSet (frozensets of sorted vertex-id triples, split into slice
and slab faces).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .field import FixedField

# mesh.py:100-128 face classes: (dt, di, dj) of (a, b, c) from the anchor
FACE_CLASS_NAMES = ("slice_lower", "slice_upper", "wall_h1", "wall_h2",
                    "wall_v1", "wall_v2", "wall_d1", "wall_d2",
                    "int_lower_a", "int_lower_b", "int_upper_a",
                    "int_upper_b")
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


@dataclass(frozen=True)
class CriticalFaceSet:
    """Faces flagged positive on the ORIGINAL fixed-point data."""
    slice_faces: frozenset
    slab_faces: frozenset
    scale: float = field(default=1.0, compare=False)

    @property
    def members(self) -> frozenset:
        return self.slice_faces | self.slab_faces

    def __len__(self):
        return len(self.slice_faces) + len(self.slab_faces)


def mask_to_faces(mask, H, W, T):
    hw = H * W
    sl, sb = set(), set()
    mask = np.asarray(mask).view(np.uint16)
    nz = np.flatnonzero(mask)
    bits = mask[nz]
    # class-major, anchors ascending: the insertion order of the reference's
    # build_critical_face_set (mesh.py:91-128 class order), so the sets'
    # iteration order -- which the reference's trajectory linking inherits
    # (tracking.py:80-101) -- is the same
    for c in range(12):
        offs = [dt * hw + di * W + dj for dt, di, dj in FACE_CLASS_OFFSETS[c]]
        dst = sl if c < 2 else sb
        for an in nz[(bits >> c) & 1 == 1].tolist():
            dst.add((an + offs[0], an + offs[1], an + offs[2]))
    return frozenset(sl), frozenset(sb)


def face_mask_fixed(H, W, T, u_fp, v_fp):
    """12-bit positive-face mask per anchor for integer field values
    (|values| < 2^30), computed by the device analysis kernel."""
    import torch
    u = torch.as_tensor(np.ascontiguousarray(u_fp, np.int64)).cuda()
    v = torch.as_tensor(np.ascontiguousarray(v_fp, np.int64)).cuda()
    if int(u.abs().max()) >= (1 << 30) or int(v.abs().max()) >= (1 << 30):
        raise ValueError("fixed values must satisfy |x| < 2^30")
    # integers < 2^30 are exact in float64 and S = 1 maps them to themselves
    return face_mask_float(H, W, T, u.double(), v.double(), 1.0)


def face_mask_float(H, W, T, du, dv, scale, host=True):
    import torch
    from .codec import Config, make_params
    from .field import dtype_code
    N = H * W * T
    p = make_params(H, W, T, 1.0, 1.0, 1.0, scale, 0, Config())
    codes = torch.empty(N, dtype=torch.uint8, device=du.device)
    ld = torch.empty((N + 31) // 32, dtype=torch.int32, device=du.device)
    mask = torch.empty(N, dtype=torch.int16, device=du.device)
    row = torch.empty(T * H, dtype=torch.int32, device=du.device)
    _lib.check(_lib.lib().vfcp_analyze(
        ctypes.byref(p), du.data_ptr(), dv.data_ptr(), dtype_code(du),
        codes.data_ptr(), ld.data_ptr(), mask.data_ptr(), row.data_ptr(),
        _lib.stream_ptr()), "analyze")
    if not host:
        return mask
    return mask.cpu().numpy().view(np.uint16)


def build_critical_face_set(ff: FixedField) -> CriticalFaceSet:
    """predicates.py:290-301 on the device."""
    mask = face_mask_fixed(ff.H, ff.W, ff.T, ff.u_fp, ff.v_fp)
    sl, sb = mask_to_faces(mask, ff.H, ff.W, ff.T)
    return CriticalFaceSet(sl, sb, ff.scale)
