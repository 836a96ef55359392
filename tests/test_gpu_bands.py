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
