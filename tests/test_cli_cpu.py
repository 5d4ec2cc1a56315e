"""CLI argument handling without a GPU (the parse layer of tools/geoheat.cpp:
CLI11 errors exit 2, --help exits 0) and the loud no-device failure."""
import subprocess

import pytest

from paper_1812_06060_b200 import _build


@pytest.fixture(scope="module")
def cli():
    return _build.build_cli()


def run(cli, args):
    return subprocess.run([cli] + args, capture_output=True, text=True)


def test_help_and_parse_errors(cli):
    r = run(cli, ["--help"])
    assert r.returncode == 0 and "distance" in r.stdout and "--out-format" in r.stdout
    assert run(cli, ["distance", "--help"]).returncode == 0
    assert run(cli, []).returncode == 2                                   # a subcommand is required
    assert run(cli, ["frobnicate"]).returncode == 2
    assert run(cli, ["distance"]).returncode == 2                         # --mesh is required
    assert run(cli, ["distance", "--mesh", "m.obj", "--frobnicate"]).returncode == 2
    assert run(cli, ["distance", "--mesh", "m.obj", "--gs-iters", "ten"]).returncode == 2
    assert run(cli, ["distance", "--mesh", "m.obj", "--m"]).returncode == 2
    assert run(cli, ["bench", "--mesh", "m.obj", "--threads-list", "1,x"]).returncode == 2
    assert run(cli, ["subdivide", "--mesh", "m.obj"]).returncode == 2    # --out is required


def test_bad_sources_are_invalid_configuration(cli):
    r = run(cli, ["distance", "--mesh", "m.obj", "--source", "1,abc"])
    assert r.returncode == 2 and "bad source index 'abc'" in r.stderr


def _has_gpu():
    from paper_1812_06060_b200 import geoheat
    return geoheat.device_count() > 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly(cli, tmp_path):
    m = tmp_path / "m.obj"
    m.write_text("v 0 0 0\nv 1 0 0\nv 0 1 0\nf 1 2 3\n")
    r = run(cli, ["distance", "--mesh", str(m), "--source", "0"])
    assert r.returncode == 1 and "no CUDA device" in r.stderr
