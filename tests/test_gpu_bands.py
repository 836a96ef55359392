"""Row-band analysis (bands.py): each band's sub-field with one
halo row per side, analysed on the device at the global S and tau', gives
exactly the reference's codes for the band's rows -- including integer
fields full of degenerate (SoS) faces -- and the bands tile the field."""

import numpy as np
import pytest

from conftest import load_golden
from paper_2510_25143_b200 import bands, synth
from paper_2510_25143_b200.field import device_range, scale_for
from paper_2510_25143_b200.codec import tau_from_eps

pytestmark = pytest.mark.gpu


def _band_codes(u, v, H, W, T, S, tau, world):
    out = []
    for rank in range(world):
        r0, r1 = bands.band_rows(H, rank, world)
        h0, h1 = bands.halo_rows(H, r0, r1)
        ub = np.ascontiguousarray(u.reshape(T, H, W)[:, h0:h1]).reshape(-1)
        vb = np.ascontiguousarray(v.reshape(T, H, W)[:, h0:h1]).reshape(-1)
        out.append(bands.analyze_band(ub, vb, H, W, T, r0, r1, S, tau)
                   .cpu().numpy())
    return np.concatenate(out, axis=1).reshape(-1)


@pytest.mark.parametrize("name", ["int1", "int3", "random_fourier_lorenzo",
                                  "vortex_pair_mop", "constant"])
@pytest.mark.parametrize("world", [2, 3, 5])
def test_band_codes_match_reference(name, world):
    g = load_golden(name)
    H, W, T = int(g["H"]), int(g["W"]), int(g["T"])
    if world > H:
        pytest.skip("more bands than rows")
    S, tau = float(g["scale"]), int(g["tau"])
    codes = _band_codes(g["u"], g["v"], H, W, T, S, tau, world)
    np.testing.assert_array_equal(codes, g["codes"])


@pytest.mark.parametrize("world", [2, 4, 7])
def test_band_codes_match_whole_field_large(world):
    H, W, T, u, v = synth.generate(1, 515, 384, 4)
    lo, hi, ma = device_range(u, v)
    S = scale_for(ma)
    tau = tau_from_eps(1e-3 * (hi - lo), S)
    whole = bands.analyze_band(u, v, H, W, T, 0, H, S, tau).cpu().numpy()
    codes = _band_codes(u, v, H, W, T, S, tau, world)
    np.testing.assert_array_equal(codes, whole.reshape(-1))
    # per-band ranges reduce to the global one (what reduce_range sums up)
    rng = []
    for rank in range(world):
        r0, r1 = bands.band_rows(H, rank, world)
        rng.append(device_range(
            np.ascontiguousarray(u.reshape(T, H, W)[:, r0:r1]).reshape(-1),
            np.ascontiguousarray(v.reshape(T, H, W)[:, r0:r1]).reshape(-1)))
    assert (min(r[0] for r in rng), max(r[1] for r in rng),
            max(r[2] for r in rng)) == (lo, hi, ma)


def _rows(a, T, H, W, r0, r1):
    return np.ascontiguousarray(a.reshape(T, H, W)[:, r0:r1]).reshape(-1)


@pytest.mark.parametrize("world", [2, 3, 6])
def test_band_face_masks_and_flip_counts(world):
    """Band masks tile the whole-field mask (and the reference's face set on
    a golden field); per-band flipped-face counts between an original and
    a perturbed reconstruction sum to verify()'s fc_t / fc_s."""
    import torch
    from paper_2510_25143_b200 import FieldSeries, verify
    from paper_2510_25143_b200.predicates import face_mask_float
    g = load_golden("int3")
    H, W, T = int(g["H"]), int(g["W"]), int(g["T"])
    S = float(g["scale"])
    whole = face_mask_float(H, W, T, torch.as_tensor(g["u"]).cuda().double(),
                            torch.as_tensor(g["v"]).cuda().double(), S,
                            host=False).view(T, H, W)
    ref = np.zeros(H * W * T, np.uint16)
    ref[g["mask_anchor"]] = g["mask_bits"]
    assert np.array_equal(whole.cpu().numpy().view(np.uint16).reshape(-1), ref)
    world = min(world, H)
    parts = []
    for rank in range(world):
        r0, r1 = bands.band_rows(H, rank, world)
        h0, h1 = bands.halo_rows(H, r0, r1)
        parts.append(bands.face_mask_band(_rows(g["u"], T, H, W, h0, h1),
                                          _rows(g["v"], T, H, W, h0, h1),
                                          H, W, T, r0, r1, S))
    assert torch.equal(torch.cat(parts, dim=1), whole)

    H, W, T, u, v = synth.generate(1, 200, 160, 4)
    rng = np.random.default_rng(5)
    ur = (u + rng.normal(0, 2e-3, u.shape)).astype(np.float32)
    vr = (v + rng.normal(0, 2e-3, v.shape)).astype(np.float32)
    S = scale_for(max(device_range(u, v)[2], device_range(ur, vr)[2]))
    counts = [0, 0]
    for rank in range(world):
        r0, r1 = bands.band_rows(H, rank, world)
        h0, h1 = bands.halo_rows(H, r0, r1)
        ma_ = bands.face_mask_band(_rows(u, T, H, W, h0, h1),
                                   _rows(v, T, H, W, h0, h1), H, W, T, r0, r1, S)
        mb_ = bands.face_mask_band(_rows(ur, T, H, W, h0, h1),
                                   _rows(vr, T, H, W, h0, h1), H, W, T, r0, r1, S)
        ct, cs = bands.flipped_faces(ma_, mb_)
        counts[0] += ct
        counts[1] += cs
    rep = verify(FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v),
                 FieldSeries(H, W, T, 1.0, 1.0, 1.0, ur, vr), scale=S)
    assert tuple(counts) == (rep.fc_t, rep.fc_s)
    assert rep.fc_t + rep.fc_s > 0


def test_face_mask_one_row_and_empty_bands():
    """bands of one row (world == H) and empty bands (world > H)
    analyse with the halo row above and give the whole-field mask."""
    import torch
    from paper_2510_25143_b200 import bands, synth
    from paper_2510_25143_b200.field import device_range, scale_for
    from paper_2510_25143_b200.predicates import face_mask_float
    H, W, T, u, v = synth.generate(1, 6, 40, 3)
    S = scale_for(device_range(u, v)[2])
    whole = face_mask_float(H, W, T, torch.as_tensor(u).cuda(),
                            torch.as_tensor(v).cuda(), S, host=False).view(T, H, W)
    for world in (H, H + 3):
        parts = []
        for rank in range(world):
            r0, r1 = bands.band_rows(H, rank, world)
            h0, h1 = bands.halo_rows(H, r0, r1)
            m = bands.face_mask_band(_rows(u, T, H, W, h0, h1),
                                     _rows(v, T, H, W, h0, h1), H, W, T, r0, r1, S)
            assert m.shape == (T, max(0, r1 - r0), W)
            parts.append(m)
        assert torch.equal(torch.cat(parts, dim=1), whole)
