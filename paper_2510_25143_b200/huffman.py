"""Canonical Huffman coding over a fixed integer alphabet.

Same blob layout and bytes as the reference (huffman.py:16,101-149):
``<IQQ`` (alphabet, symbol count, bit count) + one length byte per symbol +
MSB-first code bits.  ``encode`` runs on the host (csrc/huffman.cpp,
multi-threaded packing); ``encode_device`` packs a device symbol array on
the GPU (csrc/huffman_gpu.cu: histogram and bit packing on the device, the
code lengths on the host) and copies only the packed bytes back.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib

_HDR = struct.Struct("<IQQ")
MAX_CODE_LEN = 60


def _sym_view(symbols):
    a = np.ascontiguousarray(symbols)
    if a.dtype in (np.uint8, np.uint16, np.uint32):
        return a, a.dtype.itemsize
    if a.dtype in (np.int8, np.int16, np.int32):
        if a.size and int(a.min()) < 0:
            raise ValueError("negative symbol")
        u = a.view({1: np.uint8, 2: np.uint16, 4: np.uint32}[a.dtype.itemsize])
        return u, a.dtype.itemsize
    a = a.astype(np.int64)
    if a.size and int(a.min()) < 0:
        raise ValueError("negative symbol")
    return a, 8


def code_lengths(counts) -> np.ndarray:
    """huffman.py:21-48."""
    counts = np.ascontiguousarray(counts, dtype=np.int64)
    lens = np.zeros(counts.size, dtype=np.uint8)
    rc = _lib.lib().vfcp_huff_lengths(counts.ctypes.data, counts.size,
                                      lens.ctypes.data)
    if rc != 0:
        raise ValueError(f"code length exceeds {MAX_CODE_LEN}")
    return lens


def encode(symbols, alphabet_size: int) -> bytes:
    """Encode symbols in [0, alphabet_size) into a self-describing blob."""
    a, sb = _sym_view(symbols)
    n = a.size
    L = _lib.lib()
    counts = np.zeros(alphabet_size, dtype=np.int64)
    if n:
        _lib.check(L.vfcp_huff_count(a.ctypes.data, sb, n, alphabet_size,
                                     counts.ctypes.data), "huffman count")
    lens = code_lengths(counts)
    total_bits = int((counts * lens.astype(np.int64)).sum())
    out = np.zeros((total_bits + 7) // 8, dtype=np.uint8)
    if n:
        bits = ctypes_i64()
        _lib.check(L.vfcp_huff_pack(a.ctypes.data, sb, n, lens.ctypes.data,
                                    alphabet_size, out.ctypes.data, out.size,
                                    bits.ref(), _lib.host_threads()),
                   "huffman pack")
    return _HDR.pack(alphabet_size, n, total_bits) + lens.tobytes() + out.tobytes()


_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max(1, min(8, _lib.host_threads())))
    return _POOL


_STEP = 1 << 25


def host_copy(dst: np.ndarray, src: np.ndarray) -> None:
    """dst[:] = src for large byte arrays, split over host threads (numpy
    releases the GIL for the copies; a fresh destination's first-touch page
    faults are taken in parallel too)."""
    n = src.size
    if n <= _STEP:
        dst[:] = src
        return

    def part(o):
        dst[o:o + _STEP] = src[o:o + _STEP]
    list(_pool().map(part, range(0, n, _STEP)))


class PendingBlob:
    """A device-packed section on its way to page-locked host memory: header
    and packed bits land in one pinned buffer, and result() is a memoryview
    of it (no second copy of a section of hundreds of megabytes; the buffer
    returns to torch's caching host allocator when the section is dropped)."""

    def __init__(self, nbytes, host, words, event):
        self._nbytes = nbytes
        self._host, self._words, self._event = host, words, event

    def result(self) -> memoryview:
        self._event.synchronize()
        blob = memoryview(self._host.numpy())[:self._nbytes]
        self._host = self._words = None
        return blob


def encode_device_many(sections) -> list:
    """encode() of several CUDA uint8 / uint16 tensors, given as
    (symbols, alphabet_size, window_base[, counts]) (window_base: first symbol
    of the shared-memory histogram window, the symbols' mode; counts: the
    symbols' device histogram when the caller already has it -- the
    frame-streamed compress counts each frame as it is encoded).  All
    histograms run
    before the one host synchronisation (code lengths are built on the
    host), then every section is packed and copied to pinned memory
    asynchronously: the returned PendingBlob.result()s give the bytes."""
    import torch
    L = _lib.lib()
    st = _lib.stream_ptr()
    counts = []
    for sec in sections:
        sym, alpha, base = sec[:3]
        if len(sec) > 3 and sec[3] is not None:
            counts.append(sec[3])
            continue
        c = torch.zeros(alpha, dtype=torch.int64, device=sym.device)
        if sym.numel():
            _lib.check(L.vfcp_huff_hist_dev(sym.data_ptr(), sym.element_size(),
                                            int(sym.numel()), alpha, base,
                                            c.data_ptr(), st),
                       "huffman histogram")
        counts.append(c)
    counts = [c.cpu().numpy() for c in counts]   # one synchronisation
    out = []
    side = torch.cuda.Stream()
    for sec, counts_h in zip(sections, counts):
        sym, alpha = sec[0], sec[1]
        n = int(sym.numel())
        lens = code_lengths(counts_h)
        total_bits = int((counts_h * lens.astype(np.int64)).sum())
        n_words = max(1, (total_bits + 31) // 32)
        words = torch.empty(n_words, dtype=torch.int32, device=sym.device)
        if n:
            _lib.check(L.vfcp_huff_pack_dev(sym.data_ptr(), sym.element_size(),
                                            n, lens.ctypes.data, alpha,
                                            words.data_ptr(), n_words, st),
                       "huffman pack (device)")
        head = _HDR.pack(alpha, n, total_bits) + lens.tobytes()
        h = torch.empty(len(head) + 4 * n_words, dtype=torch.uint8,
                        pin_memory=True)
        h.numpy()[:len(head)] = np.frombuffer(head, dtype=np.uint8)
        # the copy goes to a side stream: the next section's pack kernels
        # run under it
        packed = torch.cuda.Event()
        packed.record()
        side.wait_event(packed)
        with torch.cuda.stream(side):
            h[len(head):].copy_(words.view(torch.uint8), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
        words.record_stream(side)
        out.append(PendingBlob(len(head) + (total_bits + 7) // 8, h, words, ev))
    return out


def encode_device(symbols, alphabet_size: int, window_base: int = 0):
    """encode() of a CUDA uint8 / uint16 tensor: the same bytes.

    window_base: first symbol of the shared-memory histogram window (the
    symbols' mode; radius - 4096 for the residual stream)."""
    return encode_device_many([(symbols, alphabet_size, window_base)])[0].result()



def alphabet_of(blob) -> int:
    """The alphabet size recorded in a section's header."""
    return _HDR.unpack_from(memoryview(blob), 0)[0]


def decode(blob, out_dtype=np.int64) -> np.ndarray:
    """Inverse of encode(); raises ValueError on a corrupt stream."""
    blob = memoryview(blob)
    alphabet, n_symbols, total_bits = _HDR.unpack_from(blob, 0)
    off = _HDR.size
    lens = np.frombuffer(blob, dtype=np.uint8, count=alphabet, offset=off)
    off += alphabet
    out = np.empty(n_symbols, dtype=out_dtype)
    if n_symbols == 0:
        return out
    data = np.frombuffer(blob, dtype=np.uint8,
                         count=(total_bits + 7) // 8, offset=off)
    lens = np.ascontiguousarray(lens)
    data = np.ascontiguousarray(data)
    rc = _lib.lib().vfcp_huff_unpack(data.ctypes.data, total_bits,
                                     lens.ctypes.data, alphabet, n_symbols,
                                     out.ctypes.data, out.dtype.itemsize)
    if rc != 0:
        raise ValueError("corrupt entropy stream")
    return out


def decode_device(blob, out_dtype=np.uint16):
    """decode() into a CUDA tensor (uint8 / uint16): the packed bits go to
    the device and are decoded there (csrc/huffman_gpu.cu); a stream the
    sequential decoder would reject is decoded on the host, which raises
    the reference's error."""
    import torch
    blob = memoryview(blob)
    alphabet, n_symbols, total_bits = _HDR.unpack_from(blob, 0)
    off = _HDR.size
    tdt = {np.uint8: torch.uint8, np.uint16: torch.uint16}[np.dtype(out_dtype).type]
    if n_symbols == 0:
        return torch.empty(0, dtype=tdt, device="cuda")
    lens = np.ascontiguousarray(
        np.frombuffer(blob, dtype=np.uint8, count=alphabet, offset=off))
    off += alphabet
    nbytes = (total_bits + 7) // 8
    n_words = (total_bits + 31) // 32 + 2
    hw = torch.empty(n_words, dtype=torch.int32, pin_memory=True)
    hb = hw.numpy().view(np.uint8)
    # (hundreds of megabytes: the copy is split over the host threads)
    host_copy(hb[:nbytes],
              np.frombuffer(blob, dtype=np.uint8, count=nbytes, offset=off))
    hb[nbytes:] = 0
    words = hw.cuda(non_blocking=True)
    out = torch.empty(n_symbols, dtype=tdt, device="cuda")
    L = _lib.lib()
    rc = L.vfcp_huff_unpack_dev(words.data_ptr(), n_words, total_bits,
                                lens.ctypes.data, alphabet, n_symbols,
                                out.data_ptr(), out.element_size(),
                                _lib.stream_ptr())
    if rc != 0:
        return torch.from_numpy(decode(blob, out_dtype)).cuda()
    return out


class ctypes_i64:
    def __init__(self):
        import ctypes
        self.v = ctypes.c_int64(0)

    def ref(self):
        import ctypes
        return ctypes.addressof(self.v)
