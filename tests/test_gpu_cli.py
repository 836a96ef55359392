"""The CLI end to end on the GPU path (the reference's tests/test_cli.py
scenarios): gen -> compress -> decompress -> verify, absolute bounds, a
mismatched field, a corrupt archive, and `stats` (Config.stats path)."""
import numpy as np
import pytest
from click.testing import CliRunner

from paper_2510_25143_b200.cli import main

pytestmark = pytest.mark.gpu


def _kv(output):
    out = {}
    for line in output.splitlines():
        if "=" in line:
            k, v = line.split("=", 1)
            out[k] = v
    return out


@pytest.fixture()
def runner():
    return CliRunner()


@pytest.fixture()
def workspace(tmp_path, runner):
    prefix = tmp_path / "field"
    res = runner.invoke(main, ["gen", "--config", "1", "--dims", "64x64x4",
                               "--out", str(prefix)])
    assert res.exit_code == 0, res.output
    return tmp_path, prefix


def test_full_pipeline(workspace, runner):
    tmp, prefix = workspace
    arc = tmp / "field.vfcp"
    res = runner.invoke(main, ["compress", "--input", str(prefix),
                               "--out", str(arc), "--eps-rel", "0.01"])
    assert res.exit_code == 0, res.output
    kv = _kv(res.output)
    assert float(kv["cr"]) > 1.0 and float(kv["max_abs_err"]) >= 0.0
    out = tmp / "recon"
    res = runner.invoke(main, ["decompress", "--archive", str(arc),
                               "--out", str(out)])
    assert res.exit_code == 0, res.output
    rec = np.fromfile(out.with_suffix(".u.f32"), dtype="<f4")
    orig = np.fromfile(prefix.with_suffix(".u.f32"), dtype="<f4")
    assert rec.size == orig.size
    res = runner.invoke(main, ["verify", "--input", str(prefix),
                               "--archive", str(arc)])
    assert res.exit_code == 0, res.output
    kv = _kv(res.output)
    assert kv["fc_t"] == "0" and kv["fc_s"] == "0"
    assert kv["isomorphic"] == "true"
    assert int(kv["n_traj_orig"]) > 0


def test_absolute_eps(workspace, runner):
    tmp, prefix = workspace
    res = runner.invoke(main, ["compress", "--input", str(prefix),
                               "--out", str(tmp / "abs.vfcp"), "--eps", "0.05"])
    assert res.exit_code == 0, res.output
    assert float(_kv(res.output)["max_abs_err"]) <= 0.05


def test_verify_detects_mismatched_field(workspace, runner):
    tmp, prefix = workspace
    arc = tmp / "field.vfcp"
    res = runner.invoke(main, ["compress", "--input", str(prefix),
                               "--out", str(arc), "--eps-rel", "0.01"])
    assert res.exit_code == 0, res.output
    other = tmp / "other"
    res = runner.invoke(main, ["gen", "--config", "2", "--dims", "64x64x4",
                               "--out", str(other)])
    assert res.exit_code == 0, res.output
    res = runner.invoke(main, ["verify", "--input", str(other),
                               "--archive", str(arc)])
    assert res.exit_code == 2, res.output


def test_corrupt_archive_fails(workspace, runner):
    tmp, _ = workspace
    bad = tmp / "bad.vfcp"
    bad.write_bytes(b"VFCP trailing garbage")
    res = runner.invoke(main, ["decompress", "--archive", str(bad),
                               "--out", str(tmp / "y")])
    assert res.exit_code == 1
    assert "error:" in res.output


def test_stats_writes_distribution_csvs(workspace, runner):
    tmp, prefix = workspace
    pmf, runs = tmp / "pmf.csv", tmp / "runs.csv"
    res = runner.invoke(main, ["stats", "--input", str(prefix),
                               "--eps-rel", "0.01", "--pmf-out", str(pmf),
                               "--runs-out", str(runs)])
    assert res.exit_code == 0, res.output
    kv = _kv(res.output)
    assert 0.0 <= float(kv["overflow_rate"]) <= 1.0
    assert pmf.read_text().startswith("magnitude,pmf,ccdf")
    assert runs.read_text().startswith("run_length,ccdf")


def test_track_writes_trajectory_csv(workspace, runner):
    tmp, prefix = workspace
    out = tmp / "traj.csv"
    res = runner.invoke(main, ["track", "--input", str(prefix),
                               "--out", str(out)])
    assert res.exit_code == 0, res.output
    n = int(_kv(res.output)["components"])
    rows = out.read_text().strip().splitlines()
    assert rows[0] == "component,x,y,t,loop"
    assert n > 0 and len({r.split(",")[0] for r in rows[1:]}) == n
