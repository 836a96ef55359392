"""Pin the CPU oracle (oracle/) to the reference's own outputs.

tests/golden/*.npz were produced by oracle/gen_golden.py running the real
reference; here the oracle must reproduce every section bit for bit."""
import numpy as np
import pytest

from conftest import Cfg, GOLDEN, golden_names, load_golden


@pytest.mark.parametrize("name", golden_names())
def test_oracle_matches_reference_streams(name, oracle_mod):
    O = oracle_mod
    g = load_golden(name)
    H, W, T = int(g["H"]), int(g["W"]), int(g["T"])
    cfg = Cfg(g)
    s = O.compress_streams(g["u"], g["v"], H, W, T, float(g["dx"]),
                           float(g["dy"]), float(g["dt"]), float(g["eps"]),
                           cfg, relative=bool(g["relative"]), want_mask=True)
    assert s["scale"] == float(g["scale"])
    assert s["tau"] == int(g["tau"])
    assert s["eps"] == float(g["eps_abs"])
    np.testing.assert_array_equal(s["xi"], g["xi"])
    np.testing.assert_array_equal(s["codes"], g["codes"])
    np.testing.assert_array_equal(np.packbits(s["ld"]), g["ld"])
    anchors = np.flatnonzero(s["mask"])
    np.testing.assert_array_equal(anchors, g["mask_anchor"])
    np.testing.assert_array_equal(s["mask"][anchors], g["mask_bits"])
    np.testing.assert_array_equal(s["modes"], g["modes"])
    np.testing.assert_array_equal(s["qd"], g["qd"])
    np.testing.assert_array_equal(s["ll"], g["ll"])
    if g["recon"].size:
        np.testing.assert_array_equal(
            s["recon"].reshape(2, -1), g["recon"].astype(np.int64))
        rec = O.decompress_streams(H, W, T, float(g["dx"]), float(g["dy"]),
                                   float(g["dt"]), s["scale"], s["tau"], cfg,
                                   s["codes"], s["qd"], s["ll"], s["modes"])
        np.testing.assert_array_equal(rec.reshape(2, -1),
                                      g["recon"].astype(np.int64))


@pytest.fixture(scope="module")
def prim():
    z = np.load(GOLDEN / "primitives.npz")
    return {k: z[k] for k in z.files}


def test_sos_face_predicate(prim, oracle_mod):
    L = oracle_mod.lib()
    for row in prim["sos"]:
        ua, va, ub, vb, uc, vc, a, b, c, res = (int(x) for x in row)
        assert L.or_face_positive(ua, va, ub, vb, uc, vc, a, b, c) == res


def test_orientation_sos(prim, oracle_mod):
    L = oracle_mod.lib()
    for row in prim["orient"]:
        x0, y0, x1, y1, x2, y2, i0, i1, i2, res = (int(x) for x in row)
        assert L.or_sos_sign(x0, y0, x1, y1, x2, y2, i0, i1, i2) == res


def test_face_bound(prim, oracle_mod):
    L = oracle_mod.lib()
    for row in prim["face_eb"]:
        u0, u1, u2, v0, v1, v2, res = (int(x) for x in row)
        assert L.or_face_eb(u0, v0, u1, v1, u2, v2) == res


def test_eb_ladder(prim, oracle_mod):
    for xi, tau, code in prim["ladder"]:
        assert oracle_mod.quantize_eb(int(xi), int(tau)) == int(code)
    for tau, vec in zip(prim["ladder_vec_taus"], prim["ladder_vec"]):
        codes, _ = oracle_mod.codes_from_xi(prim["ladder_vec_xi"], int(tau))
        np.testing.assert_array_equal(codes, vec)


def test_rha_bilinear_sl(prim, oracle_mod):
    L = oracle_mod.lib()
    for x, r in zip(prim["rha_x"], prim["rha"]):
        assert L.or_rha(float(x)) == int(r)
    fu = np.ascontiguousarray(prim["bil_frame"])
    fv = np.ascontiguousarray(prim["bil_frame_v"])
    H, W = fu.shape
    for (a, b), r in zip(prim["bil_pts"], prim["bil"]):
        assert L.or_bilinear(fu, H, W, float(a), float(b)) == int(r)
    out = np.zeros(2)
    for cfl, i, j, fi, fj in prim["sl"]:
        L.or_sl_departure(fu, fv, H, W, int(i), int(j), cfl, cfl * 0.7, 2.0,
                          32, out)
        assert out[0] == fi and out[1] == fj
