"""CLI and raw I/O on the host (cli.py / field.py:103-136 of the reference):
argument handling, file layout and errors that fail before any device work,
and residual_stats against the reference's own outputs
(tests/golden/residual_stats.npz, oracle/gen_residual_golden.py)."""
from pathlib import Path

import numpy as np
import pytest
from click.testing import CliRunner

from paper_2510_25143_b200 import Config, FieldError, FieldSeries
from paper_2510_25143_b200.cli import main
from paper_2510_25143_b200.field import load_meta, load_raw, save_raw
from paper_2510_25143_b200.tracking import residual_stats

GOLDEN = Path(__file__).parent / "golden" / "residual_stats.npz"


@pytest.fixture()
def runner():
    return CliRunner()


@pytest.fixture()
def workspace(tmp_path, runner):
    prefix = tmp_path / "field"
    res = runner.invoke(main, ["gen", "--config", "1", "--dims", "24x20x3",
                               "--out", str(prefix)])
    assert res.exit_code == 0, res.output
    return tmp_path, prefix


def test_gen_writes_components_and_sidecar(workspace):
    _, prefix = workspace
    n = 24 * 20 * 3
    for suffix in (".u.f32", ".v.f32"):
        assert prefix.with_suffix(suffix).stat().st_size == 4 * n
    meta = load_meta(prefix.with_suffix(".json"))
    assert (meta["H"], meta["W"], meta["T"]) == (24, 20, 3)
    assert (meta["dx"], meta["dy"], meta["dt"]) == (1.0, 1.0, 1.0)


def test_bad_dims_fails(runner, tmp_path):
    res = runner.invoke(main, ["gen", "--config", "2", "--dims", "16by16",
                               "--out", str(tmp_path / "x")])
    assert res.exit_code == 1
    assert "error:" in res.output


def test_eps_flags_mutually_exclusive(workspace, runner):
    tmp, prefix = workspace
    for extra in ([], ["--eps", "0.1", "--eps-rel", "0.01"]):
        res = runner.invoke(main, ["compress", "--input", str(prefix),
                                   "--out", str(tmp / "a.vfcp")] + extra)
        assert res.exit_code == 1
        assert "exactly one of --eps / --eps-rel" in res.output


def test_missing_input_fails(runner, tmp_path):
    res = runner.invoke(main, ["compress", "--input", str(tmp_path / "nope"),
                               "--out", str(tmp_path / "a.vfcp"),
                               "--eps-rel", "0.01"])
    assert res.exit_code == 1
    assert "missing field file" in res.output


def test_cli_defaults_mirror_config(runner):
    cfg = Config()
    cmd = main.commands["compress"]
    opts = {p.name: p.default for p in cmd.params}
    for name in ("predictor", "bx", "by", "stride", "theta", "lam", "radius",
                 "d_max", "n_max", "backend"):
        assert opts[name] == getattr(cfg, name), name


def test_raw_round_trip_and_size_check(tmp_path):
    rng = np.random.default_rng(0)
    H, W, T = 5, 7, 2
    u = rng.standard_normal(H * W * T).astype(np.float32)
    v = rng.standard_normal(H * W * T).astype(np.float32)
    f = FieldSeries(H, W, T, 0.5, 2.0, 1.0, u, v)
    up, vp, mp = tmp_path / "a.u.f32", tmp_path / "a.v.f32", tmp_path / "a.json"
    save_raw(f, up, vp, mp)
    m = load_meta(mp)
    g = load_raw(up, vp, m["H"], m["W"], m["T"], m["dx"], m["dy"], m["dt"])
    np.testing.assert_array_equal(g.u, u)
    np.testing.assert_array_equal(g.v, v)
    assert (g.dx, g.dy, g.dt) == (0.5, 2.0, 1.0)
    with pytest.raises(FieldError, match=r"expected 280 bytes \(70 float32\), got 276"):
        vp.write_bytes(vp.read_bytes()[:-4])
        load_raw(up, vp, H, W, T)
    mp.write_text('{"H": 5, "W": 7}')
    with pytest.raises(FieldError, match="metadata sidecar missing 'T'"):
        load_meta(mp)


def test_residual_stats_matches_reference():
    g = np.load(GOLDEN)
    names = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_sym")})
    assert names
    for name in names:
        r = residual_stats(g[f"{name}_sym"], int(g[f"{name}_radius"]))
        np.testing.assert_array_equal(r.folded_pmf, g[f"{name}_pmf"])
        np.testing.assert_array_equal(r.tail_ccdf, g[f"{name}_ccdf"])
        assert r.overflow_rate == float(g[f"{name}_ov"])
        np.testing.assert_array_equal(r.run_lengths, g[f"{name}_runs"])
        np.testing.assert_array_equal(r.run_ccdf, g[f"{name}_run_ccdf"])
        assert r.run_mean == float(g[f"{name}_run_mean"])
        np.testing.assert_array_equal(
            [r.run_percentiles[q] for q in (75, 80, 85, 90)], g[f"{name}_pct"])


def test_residual_stats_csv(tmp_path):
    s = residual_stats(np.array([8, 8, 9, 0]), 8)
    pmf, runs = tmp_path / "pmf.csv", tmp_path / "runs.csv"
    s.write_pmf_csv(pmf)
    s.write_runs_csv(runs)
    assert pmf.read_text().splitlines()[0] == "magnitude,pmf,ccdf"
    assert runs.read_text().startswith("run_length,ccdf")


def test_track_missing_input_fails(runner, tmp_path):
    res = runner.invoke(main, ["track", "--input", str(tmp_path / "nope"),
                               "--out", str(tmp_path / "t.csv")])
    assert res.exit_code == 1
    assert "missing field file" in res.output
    assert not (tmp_path / "t.csv").exists()


def test_track_requires_out(runner, tmp_path):
    res = runner.invoke(main, ["track", "--input", str(tmp_path / "f")])
    assert res.exit_code == 2          # click usage error, as the reference
