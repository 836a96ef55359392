"""CPU-side checks: the C-ABI library loads and exports every declared
symbol, and the host pieces of the codec (archive container, Huffman
backend, ladder) reproduce the reference's bytes on the golden vectors."""
import re
import zlib
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN, golden_names, load_golden

ROOT = Path(__file__).resolve().parents[1]


def test_library_exports_header_symbols():
    from paper_2510_25143_b200 import _lib
    L = _lib.lib()
    hdr = (ROOT / "include" / "vfcp_b200.h").read_text()
    names = set(re.findall(r"\b(vfcp_[a-z0-9_]+)\s*\(", hdr))
    assert names, "no declarations parsed"
    for n in sorted(names):
        assert hasattr(L, n), n
    assert set(_lib.EXPORTED) == names
    assert L.vfcp_version() == 1


def _sections(blob):
    from paper_2510_25143_b200 import Archive
    return Archive.from_bytes(bytes(blob))


@pytest.mark.parametrize("name", golden_names())
def test_archive_container_roundtrip(name):
    g = load_golden(name)
    for key in ("archive", "archive_identity"):
        blob = bytes(g[key])
        a = _sections(blob)
        assert a.to_bytes() == blob
        assert a.scale == float(g["scale"]) and a.tau_prime == int(g["tau"])


@pytest.mark.parametrize("name", golden_names())
def test_host_huffman_reproduces_reference_sections(name):
    from paper_2510_25143_b200 import huffman
    g = load_golden(name)
    a = _sections(g["archive"])
    assert huffman.encode(g["codes"], 32) == a.q_xi
    assert huffman.encode(g["qd"], 2 * int(g["radius"])) == a.q_d
    np.testing.assert_array_equal(huffman.decode(a.q_xi), g["codes"])
    np.testing.assert_array_equal(huffman.decode(a.q_d), g["qd"])
    assert np.packbits(g["modes"].reshape(-1)).tobytes() == a.mode_bitmap
    assert g["ll"].astype("<i8").tobytes() == a.lossless_stream
    assert g["ld"].tobytes() == a.l_d


def test_huffman_properties():
    from paper_2510_25143_b200 import huffman
    rng = np.random.default_rng(0)
    for n, alpha in ((1, 4), (2, 2), (1000, 7), (300000, 65536)):
        s = rng.integers(0, alpha, n)
        s = np.where(rng.random(n) < 0.9, s % 3, s)
        blob = huffman.encode(s, alpha)
        np.testing.assert_array_equal(huffman.decode(blob), s)
    assert huffman.decode(huffman.encode(np.zeros(0, np.int64), 5)).size == 0
    import struct
    blob = huffman.encode(np.arange(50) % 7, 7)
    alpha, n, bits = struct.unpack_from("<IQQ", blob, 0)
    # a stream that does not end exactly at its bit count is corrupt
    bad = struct.pack("<IQQ", alpha, n, bits + 1) + blob[20:] + b"\0"
    with pytest.raises(ValueError):
        huffman.decode(bad)
    bad = struct.pack("<IQQ", alpha, n + 3, bits) + blob[20:]
    with pytest.raises(ValueError):
        huffman.decode(bad)


def test_ladder_and_tau(oracle_mod):
    from paper_2510_25143_b200 import quantize_eb, tau_from_eps
    z = np.load(GOLDEN / "primitives.npz")
    for xi, tau, code in z["ladder"]:
        assert quantize_eb(int(xi), int(tau)) == int(code)
    assert tau_from_eps(0.0, 1.0) == 0
    assert tau_from_eps(1.0, 2.0 ** 20) == 2 ** 20 - 1


def test_config_validation():
    from paper_2510_25143_b200 import Config
    with pytest.raises(ValueError):
        Config(predictor="nope")
    with pytest.raises(ValueError):
        Config(backend="zstd")
    assert Config().mop.r_meta == 1.0 / 2048


def test_archive_errors():
    from paper_2510_25143_b200 import Archive
    g = load_golden("vortex_small")
    blob = bytes(g["archive"])
    with pytest.raises(ValueError):
        Archive.from_bytes(b"nope" + blob[4:])
    with pytest.raises(ValueError):
        Archive.from_bytes(blob[:-5])
    bad = bytearray(blob)
    bad[4] = 9
    with pytest.raises(ValueError):
        Archive.from_bytes(bytes(bad))


def test_host_range_exact():
    """vfcp_host_range (the streamed path's early value range) equals
    numpy's min / max / max|x| on both dtypes, any length and thread count."""
    from paper_2510_25143_b200 import _lib
    rng = np.random.default_rng(11)
    for dtype, code in ((np.float32, _lib.VFCP_F32), (np.float64, _lib.VFCP_F64)):
        for n, nt in ((1, 4), (15, 1), (4097, 3), (2 * (1 << 20) + 3, 8)):
            u = (rng.standard_normal(n) * 3).astype(dtype)
            v = (rng.standard_normal(n) * 5 - 1).astype(dtype)
            out = np.zeros(3)
            _lib.check(_lib.lib().vfcp_host_range(
                u.ctypes.data, v.ctypes.data, code, n, nt, out.ctypes.data),
                "host range")
            assert out[0] == min(u.min(), v.min())
            assert out[1] == max(u.max(), v.max())
            assert out[2] == max(np.abs(u).max(), np.abs(v).max())
    out = np.zeros(3)
    assert _lib.lib().vfcp_host_range(None, None, 0, 0, 1, out.ctypes.data) != 0
