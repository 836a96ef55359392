"""ctypes binding of the C ABI in include/vfcp_b200.h (libvfcp_b200.so).

This is the only way the package reaches the device: there is no CPU
fallback.  If the library is missing the package raises on first use.
Device buffers are torch CUDA tensors (plumbing only); their data pointers
and torch's current CUDA stream are passed straight through.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = _HERE / "_lib" / (
    "libvfcp_b200_debug.so" if os.environ.get("VFCP_DEBUG_LIB") else
    "libvfcp_b200.so")

VFCP_F32, VFCP_F64 = 0, 1
PRED_INDEX = {"mop": 0, "lorenzo": 1, "sl": 2}


class vfcp_params(ctypes.Structure):
    _fields_ = [
        ("H", ctypes.c_int32), ("W", ctypes.c_int32), ("T", ctypes.c_int32),
        ("dx", ctypes.c_double), ("dy", ctypes.c_double),
        ("dt", ctypes.c_double), ("scale", ctypes.c_double),
        ("tau", ctypes.c_int64), ("predictor", ctypes.c_int32),
        ("bx", ctypes.c_int32), ("by", ctypes.c_int32),
        ("stride", ctypes.c_int32), ("radius", ctypes.c_int32),
        ("n_max", ctypes.c_int32), ("lam", ctypes.c_double),
        ("theta", ctypes.c_double), ("d_max", ctypes.c_double),
    ]


_lib = None
_P = ctypes.c_void_p
_I = ctypes.c_int
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_PP = ctypes.POINTER(vfcp_params)

_SIGS = {
    "vfcp_last_error": (ctypes.c_char_p, []),
    "vfcp_version": (_I, []),
    "vfcp_launch_count": (_I64, []),
    "vfcp_prof_enable": (_I, [_I]),
    "vfcp_prof_collect": (_I, [_P, _P, _I]),
    "vfcp_value_range": (_I, [_P, _P, _I, _I64, _P, _P]),
    "vfcp_analyze": (_I, [_PP, _P, _P, _I, _P, _P, _P, _P, _P]),
    "vfcp_qd_offsets": (_I, [_PP, _P, _P, _P, _P]),
    "vfcp_encode": (_I, [_PP, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vfcp_encode_host": (_I, [_PP, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P, _P]),
    "vfcp_host_range": (_I, [_P, _P, _I, _I64, _I, _P]),
    "vfcp_value_range_part": (_I, [_P, _P, _I, _I64, _P, _I, _P]),
    "vfcp_analyze_slab": (_I, [_PP, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P,
                               _I64, _P, _P, _P]),
    "vfcp_qd_offsets_upto": (_I, [_PP, _I, _P, _P, _P, _P]),
    "vfcp_encode_stream_begin": (_I, [_PP, _P, _P, _I, _P, _P, _P, _P, _P,
                                      _P, _P]),
    "vfcp_encode_stream_frame": (_I, [_P, _I]),
    "vfcp_encode_stream_end": (_I, [_P, _P]),
    "vfcp_row_offsets": (_I, [_P, _I64, _P, _P, _P]),
    "vfcp_encode_ll": (_I, [_PP, _P, _P, _I, _P, _P, _P, _P, _P, _P, _P]),
    "vfcp_decode_prepare": (_I, [_PP, _P, _P, _P, _I64, _P, _P, _P, _P, _P,
                                 _P, _P]),
    "vfcp_decode": (_I, [_PP, _P, _P, _I64, _P, _I64, _P, _P, _P, _P, _P,
                         _P, _P, _P]),
    "vfcp_decode_host": (_I, [_PP, _P, _P, _I64, _P, _I64, _P, _P, _P, _P,
                              _P, _P, _P, _P]),
    "vfcp_huff_lengths": (_I, [_P, _I32, _P]),
    "vfcp_huff_count": (_I, [_P, _I, _I64, _I32, _P]),
    "vfcp_huff_pack": (_I, [_P, _I, _I64, _P, _I32, _P, _I64, _P, _I]),
    "vfcp_huff_unpack": (_I, [_P, _I64, _P, _I32, _I64, _P, _I]),
    "vfcp_huff_hist_dev": (_I, [_P, _I, _I64, _I32, _I32, _P, _P]),
    "vfcp_huff_pack_dev": (_I, [_P, _I, _I64, _P, _I32, _P, _I64, _P]),
    "vfcp_huff_unpack_dev": (_I, [_P, _I64, _I64, _P, _I32, _I64, _P, _I, _P]),
}

EXPORTED = tuple(_SIGS)

# launch classes of vfcp_prof_collect (capi.cu KClass): "analyze" the split
# analysis (cube test + exact pass), "enc_block" / "dec_block" the per-block
# frame kernels, "bs_chain" the block-scan kernel (chain + interior passes),
# "scan" the prefix counts; "mop" / "encode" / "decode" the generic path
KERNEL_CLASSES = ("range", "analyze", "scan", "mop", "encode", "ll_write",
                  "decode_rows", "decode_ll", "decode", "aux", "enc_block",
                  "dec_block", "bs_chain")


def prof_enable(on=True):
    lib().vfcp_prof_enable(1 if on else 0)


def prof_collect():
    """{class: (total ms, launches)} since prof_enable (synchronising)."""
    n = len(KERNEL_CLASSES)
    ms = np.zeros(n, np.float64)
    cnt = np.zeros(n, np.int64)
    check(lib().vfcp_prof_collect(ms.ctypes.data, cnt.ctypes.data, n),
          "prof_collect")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_CLASSES)}


def launch_count() -> int:
    return int(lib().vfcp_launch_count())


class VfcpError(RuntimeError):
    pass


def lib():
    """Load libvfcp_b200.so (built by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise VfcpError(
                f"{LIB_PATH} missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(rc: int, what: str):
    if rc != 0:
        msg = lib().vfcp_last_error().decode(errors="replace")
        if rc in (-1, -4):   # VFCP_EINVAL, VFCP_ECORRUPT: the reference's ValueError
            raise ValueError(f"{what}: {msg}")
        raise VfcpError(f"{what} failed ({rc}): {msg}")


def ptr(t) -> int:
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def stream_ptr():
    import torch
    return torch.cuda.current_stream().cuda_stream


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)
