"""Config.stats / CompressStats parity with the reference (codec.py:388-397)
and FieldSeries validation on device tensors (field.py:37-51).

tests/golden/compress_stats.npz holds the reference's own CompressStats
(oracle/gen_stats_golden.py ran the reference's compress with stats=True on
the golden fields): symbols, signed_indices, overflow_count,
lossless_vertices, modes and critical_faces must be identical."""
import numpy as np
import pytest

from conftest import GOLDEN, load_golden

pytestmark = pytest.mark.gpu

STATS = np.load(GOLDEN / "compress_stats.npz")
NAMES = sorted({k.split("__")[0] for k in STATS.files})


def _field_and_cfg(name, device):
    import torch
    import paper_2510_25143_b200 as vg
    g = load_golden(name)
    u, v = g["u"], g["v"]
    if device:
        u, v = torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda()
    f = vg.FieldSeries(int(g["H"]), int(g["W"]), int(g["T"]), float(g["dx"]),
                       float(g["dy"]), float(g["dt"]), u, v)
    cfg = vg.Config(predictor=str(g["predictor"]), radius=int(g["radius"]),
                    bx=int(g["bx"]), by=int(g["by"]), stride=int(g["stride"]),
                    lam=float(g["lam"]), theta=float(g["theta"]),
                    d_max=float(g["d_max"]), n_max=int(g["n_max"]), stats=True)
    return f, cfg, float(g["eps"]), bool(g["relative"])


@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("device", [False, True])
def test_compress_stats_match_reference(name, device):
    import paper_2510_25143_b200 as vg
    f, cfg, eps, rel = _field_and_cfg(name, device)
    s = vg.compress(f, eps, cfg, relative=rel).stats
    assert s is not None
    np.testing.assert_array_equal(s.symbols, STATS[f"{name}__symbols"])
    assert s.symbols.dtype == np.int32
    np.testing.assert_array_equal(s.signed_indices, STATS[f"{name}__signed"])
    assert s.signed_indices.dtype == np.int32
    assert s.overflow_count == int(STATS[f"{name}__overflow"])
    assert s.lossless_vertices == int(STATS[f"{name}__lossless"])
    np.testing.assert_array_equal(s.modes, STATS[f"{name}__modes"])
    assert s.modes.shape == STATS[f"{name}__modes"].shape
    assert s.critical_faces == int(STATS[f"{name}__faces"])


def test_no_stats_by_default():
    import paper_2510_25143_b200 as vg
    f, cfg, eps, rel = _field_and_cfg(NAMES[0], True)
    import dataclasses
    a = vg.compress(f, eps, dataclasses.replace(cfg, stats=False), relative=rel)
    assert a.stats is None


@pytest.mark.parametrize("dtype", ["float32", "float64"])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("inf")])
def test_device_nonfinite_rejected(dtype, bad):
    """field.py:48-51 on CUDA tensors: the first non-finite index is named."""
    import torch
    import paper_2510_25143_b200 as vg
    H, W, T = 6, 7, 3
    u = torch.zeros(H * W * T, dtype=getattr(torch, dtype), device="cuda")
    v = torch.ones_like(u)
    v[17] = bad
    v[40] = bad
    with pytest.raises(vg.FieldError, match=r"non-finite sample in v at index 17"):
        vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    u[5] = bad
    with pytest.raises(vg.FieldError, match=r"non-finite sample in u at index 5"):
        vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)


def test_device_bad_dims_and_lengths_rejected():
    import torch
    import paper_2510_25143_b200 as vg
    u = torch.zeros(24, device="cuda")
    with pytest.raises(vg.FieldError, match=r"dims must be >= 2, got 1x12x2"):
        vg.FieldSeries(1, 12, 2, 1.0, 1.0, 1.0, u, u)
    with pytest.raises(vg.FieldError, match="dx, dy, dt must be positive"):
        vg.FieldSeries(2, 6, 2, 0.0, 1.0, 1.0, u, u)
    with pytest.raises(vg.FieldError, match=r"component length mismatch: expected 27"):
        vg.FieldSeries(3, 3, 3, 1.0, 1.0, 1.0, u, u)


def test_device_nonfinite_through_compress():
    """compress() on a device field never sees a non-finite sample: the
    FieldSeries constructor rejects it first, as the reference's does."""
    import torch
    import paper_2510_25143_b200 as vg
    u = torch.randn(4 * 5 * 2, device="cuda")
    u[-1] = float("nan")
    with pytest.raises(vg.FieldError):
        f = vg.FieldSeries(4, 5, 2, 1.0, 1.0, 1.0, u, u.clone())
        vg.compress(f, 0.1)


WIDE = np.load(GOLDEN / "wide_codes.npz")


@pytest.mark.parametrize("tag", ["a", "b"])
def test_wide_code_alphabet_matches_reference(tag):
    """A q_xi section with an alphabet past 32 (codes 33, 40, 287, 300):
    decoded with the reference's tau >> min(code, K_MAX) rule,
    giving the reference's reconstruction or its error."""
    import paper_2510_25143_b200 as vg
    for variant in ("ok", "bad"):
        a = vg.Archive.from_bytes(WIDE[f"{tag}_{variant}_archive"].tobytes())
        err = str(WIDE[f"{tag}_{variant}_error"])
        if err:
            with pytest.raises(ValueError, match=err):
                vg.reconstruct_fixed(a)
        else:
            r = vg.reconstruct_fixed(a)
            want = WIDE[f"{tag}_{variant}_recon"]
            np.testing.assert_array_equal(r.u_fp, want[0])
            np.testing.assert_array_equal(r.v_fp, want[1])
