"""Device path vs the reference's golden vectors (bit-exact).

Every section the reference produced for the golden fields -- eb codes,
l_d, the critical-face set, modes, qd symbols, ll and the archive bytes --
must come out of the B200 kernels identically, and decompression must
reproduce the reference's fixed-point reconstruction exactly."""
import numpy as np
import pytest

from conftest import golden_names, load_golden

pytestmark = pytest.mark.gpu


def _field(g):
    import paper_2510_25143_b200 as vg
    return vg.FieldSeries(int(g["H"]), int(g["W"]), int(g["T"]),
                          float(g["dx"]), float(g["dy"]), float(g["dt"]),
                          g["u"], g["v"])


def _cfg(g, **kw):
    import paper_2510_25143_b200 as vg
    return vg.Config(predictor=str(g["predictor"]), bx=int(g["bx"]),
                     by=int(g["by"]), stride=int(g["stride"]),
                     lam=float(g["lam"]), theta=float(g["theta"]),
                     radius=int(g["radius"]), d_max=float(g["d_max"]),
                     n_max=int(g["n_max"]), **kw)


@pytest.mark.parametrize("name", golden_names())
def test_device_streams_match_reference(name):
    import paper_2510_25143_b200 as vg
    g = load_golden(name)
    f = _field(g)
    s = vg.compress_device(f, float(g["eps"]), _cfg(g),
                           relative=bool(g["relative"]), want_mask=True)
    assert s.scale == float(g["scale"])
    assert s.tau == int(g["tau"])
    assert s.eps == float(g["eps_abs"])
    np.testing.assert_array_equal(s.codes.cpu().numpy(), g["codes"])
    np.testing.assert_array_equal(s.ld.cpu().numpy(), g["ld"])
    mask = s.mask.cpu().numpy().view(np.uint16)
    anchors = np.flatnonzero(mask)
    np.testing.assert_array_equal(anchors, g["mask_anchor"])
    np.testing.assert_array_equal(mask[anchors], g["mask_bits"])
    np.testing.assert_array_equal(s.modes.cpu().numpy(),
                                  g["modes"].reshape(-1))
    np.testing.assert_array_equal(s.qd.cpu().numpy().astype(np.int32),
                                  g["qd"])
    np.testing.assert_array_equal(s.ll.cpu().numpy(), g["ll"])


@pytest.mark.parametrize("name", golden_names())
def test_archive_bytes_and_decode_match_reference(name):
    import paper_2510_25143_b200 as vg
    g = load_golden(name)
    f = _field(g)
    a = vg.compress(f, float(g["eps"]), _cfg(g), relative=bool(g["relative"]))
    assert a.to_bytes() == bytes(g["archive"])
    ai = vg.compress(f, float(g["eps"]), _cfg(g, backend="identity"),
                     relative=bool(g["relative"]))
    assert ai.to_bytes() == bytes(g["archive_identity"])
    b = vg.Archive.from_bytes(bytes(g["archive"]))
    if str(g["decode_error"]):
        with pytest.raises(ValueError, match="lossless bitmap"):
            vg.decompress(b)
        return
    r = vg.reconstruct_fixed(b)
    np.testing.assert_array_equal(r.u_fp, g["recon"][0].astype(np.int64))
    np.testing.assert_array_equal(r.v_fp, g["recon"][1].astype(np.int64))
    fs, ds = vg.decompress_with_stats(b)
    assert ds.aux_component_buffers == 4
    S = float(g["scale"])
    np.testing.assert_array_equal(fs.u, g["recon"][0].astype(np.int64) * (1.0 / S))
    np.testing.assert_array_equal(fs.v, g["recon"][1].astype(np.int64) * (1.0 / S))
    # every point within the user bound (guaranteed once eps*S >= 1/2,
    # i.e. tau' >= 0 covers the fixed-point rounding, codec.py:71-77)
    if float(g["eps_abs"]) * S < 0.5:
        return
    err = max(np.abs(fs.u - g["u"].astype(np.float64)).max(),
              np.abs(fs.v - g["v"].astype(np.float64)).max())
    assert err <= float(g["eps_abs"])


@pytest.mark.parametrize("name", ["vortex_small", "cfg1_eps0.01",
                                  "random_fourier_mop", "int3"])
def test_recon_preserves_critical_faces(name):
    """Decompressed field has exactly the original critical-face set."""
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200.predicates import face_mask_float
    import torch
    g = load_golden(name)
    f = _field(g)
    a = vg.compress(f, float(g["eps"]), _cfg(g), relative=bool(g["relative"]))
    ou, ov, _, _ = vg.decompress_device(a)
    H, W, T = f.H, f.W, f.T
    S = a.scale
    m_orig = face_mask_float(H, W, T, torch.from_numpy(g["u"]).cuda(),
                             torch.from_numpy(g["v"]).cuda(), S)
    m_rec = face_mask_float(H, W, T, ou, ov, S)
    np.testing.assert_array_equal(m_orig, m_rec)
