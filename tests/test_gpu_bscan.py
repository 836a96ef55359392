"""Block-scan chain and MoP trial vs the CPU oracle on fields that reach
every path of bscan.cuh (bit-exact).

The golden fields are small (at most 4 x 4 blocks), so these cases add:
frames with more block rows than one chain CTA holds (tagged global
handoff between CTAs) and ragged edges; tiny steps (tau' of a few units),
where residue ties are frequent on block edges and inside blocks; integer
fields with a small radius (escapes, swept blocks); vortex fields with
mixed quantisation steps and lossless vertices near critical points; and
every predictor."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _ints(H, W, T, seed, lo, hi):
    rng = np.random.default_rng(seed)
    u = rng.integers(lo, hi, H * W * T).astype(np.float32)
    v = rng.integers(lo, hi, H * W * T).astype(np.float32)
    return H, W, T, u, v


def _synth(cfg, H, W, T):
    from paper_2510_25143_b200 import synth
    return synth.generate(cfg, H, W, T)


CASES = {
    # (field, eps, relative, predictor, radius)
    "spectral_multicta_mop": (lambda: _synth(2, 300, 520, 3), 1e-3, True, "mop", 32768),
    "spectral_ragged_lorenzo": (lambda: _synth(5, 290, 333, 2), 1e-4, True, "lorenzo", 32768),
    "spectral_sl": (lambda: _synth(5, 270, 200, 3), 1e-3, True, "sl", 32768),
    "vortex_mixed_steps": (lambda: _synth(1, 320, 256, 4), 1e-2, True, "mop", 32768),
    "wake_mop": (lambda: _synth(3, 288, 256, 3), 1e-3, True, "mop", 32768),
    # tau' of a few fixed-point units: ties everywhere
    "tiny_tau_lorenzo": (lambda: _synth(2, 280, 300, 2), 2e-9, True, "lorenzo", 32768),
    "tiny_tau_mop": (lambda: _synth(5, 260, 270, 3), 4e-9, True, "mop", 32768),
    # integers, small radius: escapes and swept blocks
    "ints_radius16": (lambda: _ints(270, 300, 3, 7, -40, 41), 0.02, True, "mop", 16),
    # rows wider than one 256-chunk segment of the prefix-count kernel,
    # with escapes (and a ragged last chunk)
    "ints_wide_radius16": (lambda: _ints(40, 9000, 2, 9, -40, 41), 0.02, True, "mop", 16),
    "spectral_wide_sl": (lambda: _synth(2, 48, 8230, 2), 1e-3, True, "sl", 32768),
    # large steps: tau' in [2^28, 2^29) (the widest the block kernels take,
    # sums in int64) and just past it (the generic kernels)
    "large_tau_mop": (lambda: _synth(5, 200, 230, 3), 0.2, True, "mop", 32768),
    "large_tau_lorenzo": (lambda: _synth(2, 230, 190, 3), 0.35, True, "lorenzo", 32768),
    "huge_tau_generic": (lambda: _synth(5, 130, 150, 3), 0.6, True, "mop", 32768),
    # integers on a step of one fixed-point unit: exact reconstruction
    "ints_unit_step": (lambda: _ints(300, 260, 2, 8, -3, 4), 2.0 / 2 ** 28, False, "lorenzo", 32768),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_bscan_paths_match_oracle(name):
    import paper_2510_25143_b200 as vg
    from oracle import cpu_oracle as O
    gen, eps, rel, pred, radius = CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred, radius=radius)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    s = vg.compress_device(f, eps, cfg, relative=rel)
    ref = O.compress_streams(u, v, H, W, T, 1.0, 1.0, 1.0, eps, cfg,
                             relative=rel)
    assert s.scale == ref["scale"] and s.tau == ref["tau"]
    if name.startswith("large_tau"):
        assert 2 ** 28 <= s.tau < 2 ** 29, s.tau
    np.testing.assert_array_equal(s.codes.cpu().numpy(), ref["codes"])
    np.testing.assert_array_equal(s.modes.cpu().numpy(),
                                  ref["modes"].reshape(-1))
    np.testing.assert_array_equal(s.qd.cpu().numpy().astype(np.int32),
                                  ref["qd"])
    np.testing.assert_array_equal(s.ll.cpu().numpy(), ref["ll"])
    # decode of the same streams: the fixed-point reconstruction
    a = vg.compress(f, eps, cfg, relative=rel)
    r = vg.reconstruct_fixed(a)
    np.testing.assert_array_equal(r.u_fp, ref["recon"][0].reshape(-1))
    np.testing.assert_array_equal(r.v_fp, ref["recon"][1].reshape(-1))


@pytest.mark.parametrize("name", ["spectral_multicta_mop", "ints_radius16"])
def test_host_streaming_matches_device_streams(name):
    """compress_device(host_out=True): the symbol stream copied frame by frame
    to pinned host memory while later frames encode equals the device
    streams."""
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200 import codec
    gen, eps, rel, pred, radius = CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred, radius=radius)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    s = vg.compress_device(f, eps, cfg, relative=rel, host_out=True)
    assert s.host is not None
    d = codec.streams_to_host(vg.compress_device(f, eps, cfg, relative=rel))
    for k in ("codes", "ld", "qd", "ll", "modes"):
        np.testing.assert_array_equal(s.host[k], d[k])


@pytest.mark.parametrize("name", ["spectral_multicta_mop", "ints_radius16",
                                  "tiny_tau_mop"])
def test_device_huffman_matches_host(name):
    """huffman.encode_device (histogram + canonical-code bit packing on the
    GPU) gives the host encoder's bytes, for the eb codes and the residual
    symbols."""
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200 import huffman
    gen, eps, rel, pred, radius = CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred, radius=radius)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    s = vg.compress_device(f, eps, cfg, relative=rel)
    assert huffman.encode_device(s.codes, 32) == huffman.encode(s.codes.cpu().numpy(), 32)
    assert (huffman.encode_device(s.qd, 2 * radius, max(0, radius - 4096))
            == huffman.encode(s.qd.cpu().numpy(), 2 * radius))


@pytest.mark.parametrize("name", ["spectral_multicta_mop", "ints_radius16",
                                  "tiny_tau_mop"])
def test_device_huffman_decode(name):
    """huffman.decode_device (chunk-parallel, resynchronised decode on the
    GPU) returns the symbols of the host decoder."""
    import paper_2510_25143_b200 as vg
    from paper_2510_25143_b200 import huffman
    gen, eps, rel, pred, radius = CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred, radius=radius)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    s = vg.compress_device(f, eps, cfg, relative=rel)
    for sym, alpha, dt in ((s.codes, 32, np.uint8), (s.qd, 2 * radius, np.uint16)):
        blob = huffman.encode(sym.cpu().numpy(), alpha)
        np.testing.assert_array_equal(huffman.decode_device(blob, dt).cpu().numpy(),
                                      huffman.decode(blob, dt))
    # a truncated stream: the host decoder's error
    blob = huffman.encode(s.qd.cpu().numpy(), 2 * radius)
    with pytest.raises(ValueError):
        huffman.decode_device(blob[:-3], np.uint16)


@pytest.mark.parametrize("name", ["spectral_multicta_mop", "ints_radius16"])
def test_decompress_host_paths_agree(name, monkeypatch):
    """decompress() streams each frame's output to pinned host memory
    (vfcp_decode_host); the generic decoder (VFCP_SLOW_PATH) copies it at
    the end: both give the device decoder's output."""
    import torch
    import paper_2510_25143_b200 as vg
    gen, eps, rel, pred, radius = CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred, radius=radius)
    a = vg.compress(vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v), eps, cfg,
                    relative=rel)
    du, dv, _, _ = vg.decompress_device(a)
    fast = vg.decompress(a)
    monkeypatch.setenv("VFCP_SLOW_PATH", "1")
    slow = vg.decompress(a)
    for f in (fast, slow):
        np.testing.assert_array_equal(f.u, du.cpu().numpy())
        np.testing.assert_array_equal(f.v, dv.cpu().numpy())


VECTOR_CASES = {
    # frames of at least 1024 blocks with 16-byte rows: the four-pixel forms of
    # the interior passes (bscan.cuh bs_final_enc4 / bs_final_dec4), the
    # decoder's fast block kernel and its worklist (dec_block.cu), the vector
    # pre-passes of the decoder (decode.cu)
    "spectral_1024_mop": (lambda: _synth(5, 1024, 1040, 3), 1e-3, "mop"),
    "vortex_1056_mop": (lambda: _synth(1, 1056, 1024, 3), 1e-2, "mop"),
    "wake_1024_sl": (lambda: _synth(3, 1024, 1024, 2), 1e-3, "sl"),
    # rows that are not a multiple of 4: every vector form falls back
    "spectral_1030_lorenzo": (lambda: _synth(2, 1024, 1030, 2), 1e-3, "lorenzo"),
}


@pytest.mark.parametrize("name", sorted(VECTOR_CASES))
def test_vector_forms_match_oracle(name):
    """Streams, float64 output (the float64-only decode takes the vector
    interior) and fixed-point reconstruction vs the oracle, bit-exact."""
    import paper_2510_25143_b200 as vg
    from oracle import cpu_oracle as O
    gen, eps, pred = VECTOR_CASES[name]
    H, W, T, u, v = gen()
    cfg = vg.Config(predictor=pred)
    f = vg.FieldSeries(H, W, T, 1.0, 1.0, 1.0, u, v)
    s = vg.compress_device(f, eps, cfg, relative=True)
    ref = O.compress_streams(u, v, H, W, T, 1.0, 1.0, 1.0, eps, cfg,
                             relative=True)
    assert s.scale == ref["scale"] and s.tau == ref["tau"]
    np.testing.assert_array_equal(s.codes.cpu().numpy(), ref["codes"])
    np.testing.assert_array_equal(s.modes.cpu().numpy(),
                                  ref["modes"].reshape(-1))
    np.testing.assert_array_equal(s.qd.cpu().numpy().astype(np.int32),
                                  ref["qd"])
    np.testing.assert_array_equal(s.ll.cpu().numpy(), ref["ll"])
    a = vg.compress(f, eps, cfg, relative=True)
    du, dv, _, _ = vg.decompress_device(a)
    inv = 1.0 / ref["scale"]
    np.testing.assert_array_equal(du.cpu().numpy(),
                                  ref["recon"][0].reshape(-1).astype(np.float64) * inv)
    np.testing.assert_array_equal(dv.cpu().numpy(),
                                  ref["recon"][1].reshape(-1).astype(np.float64) * inv)
    r = vg.reconstruct_fixed(a)
    np.testing.assert_array_equal(r.u_fp, ref["recon"][0].reshape(-1))
    np.testing.assert_array_equal(r.v_fp, ref["recon"][1].reshape(-1))
