"""The CLI drop-in on the GPU: lib/geoheat_b200 run
through the shell like reference/proj/tests/test_cli.cpp drives the reference
tool — the same cases (unit square, zero ADMM iterations, exit codes,
bitwise determinism across thread flags, reference comparison, report keys,
GEOHEAT_THREADS, csv/ply outputs, bench CSV sweep, subdivide) — plus value
parity with the compiled reference's run_pipeline chain.
"""
import os
import subprocess

import numpy as np
import pytest

from paper_1812_06060_b200 import _build

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cli():
    path = _build.build_cli()
    assert os.path.exists(path)
    return path


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    assert available("reference"), "oracle/_ref/libgeoheat_ref.so missing"
    return Oracle("reference")


def run(cli, args, env=None, **kw):
    import paper_1812_06060_b200 as gh
    gh.geoheat.release_cached_memory()  # the child process needs device memory this one may cache
    e = dict(os.environ)
    e.pop("GEOHEAT_THREADS", None)
    if env:
        e.update(env)
    return subprocess.run([cli] + args, capture_output=True, env=e, **kw)


def write_mesh(gpu, ref, tmp_path, name, gen, *params):
    P, F = ref.test_mesh(gen, *params)
    path = str(tmp_path / name)
    gpu.geoheat.save_mesh(path, gpu.geoheat.build_mesh(P, F))
    return path, P, F


def read_txt(path):
    return np.array([float(x) for x in open(path).read().split()])


def report_value(text, key):
    for line in text.splitlines():
        if line.startswith(key + " = "):
            return float(line[len(key) + 3:])
    return float("nan")


def test_unit_square_edge(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "square.obj", "unit_square")
    out = str(tmp_path / "sq.txt")
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--method", "edge", "--seq", "--out", out])
    assert r.returncode == 0, r.stderr
    d = read_txt(out)
    assert d.size == 4 and d[0] == 0.0 and np.all(np.isfinite(d))


def test_zero_admm_iterations(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "square0.obj", "unit_square")
    out, rep = str(tmp_path / "sq0.txt"), str(tmp_path / "sq0.report")
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--method", "face", "--admm-iters", "0", "--seq",
                  "--out", out, "--report", rep])
    assert r.returncode == 0, r.stderr
    assert report_value(open(rep).read(), "admm_iterations") == 0.0
    assert read_txt(out).size == 4


def test_exit_codes(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "square_codes.obj", "unit_square")
    assert run(cli, ["distance", "--mesh", "/nonexistent/mesh.obj", "--source", "0"]).returncode == 1
    bad = tmp_path / "bad.obj"
    bad.write_text("v 0 0 0\nf 1 2 9\n")
    r = run(cli, ["distance", "--mesh", str(bad), "--source", "0"])
    assert r.returncode == 1 and b"OBJ parse failure at line 2" in r.stderr
    assert run(cli, ["distance", "--mesh", mesh, "--method", "bogus", "--source", "0"]).returncode == 2
    assert run(cli, ["distance", "--mesh", mesh, "--m", "-1", "--source", "0"]).returncode == 2
    r = run(cli, ["distance", "--mesh", mesh, "--source", "99"])
    assert r.returncode == 2 and b"source index 99 out of range" in r.stderr
    assert run(cli, ["distance", "--mesh", mesh, "--frobnicate"]).returncode == 2
    assert run(cli, ["distance", "--mesh", mesh, "--source", "x"]).returncode == 2
    assert run(cli, ["distance", "--mesh", mesh, "--out-format", "xml", "--out", str(tmp_path / "o")]).returncode == 2
    assert run(cli, ["distance", "--mesh", mesh, "--reference", "moon"]).returncode == 2
    assert run(cli, ["distance", "--mesh", mesh, "--device", "cpu"]).returncode == 2
    assert run(cli, ["--help"]).returncode == 0


def test_identical_flags_bitwise_identical(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "disk_det.obj", "hex_disk", 10)
    base = ["distance", "--mesh", mesh, "--source", "0", "--method", "face", "--gs-iters", "200"]
    outs = []
    for extra in (["--threads", "1"], ["--threads", "1"], ["--threads", "4"], ["--seq"]):
        p = str(tmp_path / f"det{len(outs)}.txt")
        assert run(cli, base + extra + ["--out", p]).returncode == 0
        outs.append(open(p, "rb").read())
    assert all(o == outs[0] for o in outs)


def test_reference_comparison_flat_disk(gpu, ref, cli, tmp_path):
    mesh, P, F = write_mesh(gpu, ref, tmp_path, "disk_ref.obj", "hex_disk", 25)
    rep, out = str(tmp_path / "ref.report"), str(tmp_path / "ref.txt")
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--seq", "--reference", "euclid", "--out", out,
                  "--report", rep])
    assert r.returncode == 0, r.stderr
    text = open(rep).read()
    eps = report_value(text, "mean_rel_error")
    assert np.isfinite(eps) and eps <= 0.02
    # the same metric from the reference's own oracle on our distances
    om = ref.build_mesh(P, F)
    d = read_txt(out)
    assert eps == om.mean_relative_error(d, om.analytic(0, [0]), [0])
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--reference", "dijkstra", "--report", rep,
                  "--out", out])
    assert r.returncode == 0 and "reference = dijkstra" in open(rep).read()


def test_report_echoes_configuration(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "square_rep.obj", "unit_square")
    rep = str(tmp_path / "full.report")
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0,2", "--method", "edge", "--m", "2.5", "--gs-iters", "77",
                  "--admm-iters", "3", "--mu", "50", "--eps", "1e-4", "--threads", "2", "--report", rep])
    assert r.returncode == 0, r.stderr
    text = open(rep).read()
    for key in ("method = edge", "sources = 0,2", "m = 2.5", "gs_iters = 77", "admm_iters = 3", "mu = 50",
                "eps1 = 0.0001", "eps2 = 0.0001", "threads = 2", "seq = 0"):
        assert key in text, key
    for key in ("t = ", "tau = ", "avg_edge_length = ", "init_seconds", "diffusion_seconds", "optimization_seconds",
                "integration_seconds", "total_seconds", "solver_state_bytes", "gs_iterations", "final_primal",
                "final_dual", "diffusion_e1"):
        assert key in text, key
    s = sum(report_value(text, k) for k in ("init_seconds", "diffusion_seconds", "optimization_seconds",
                                            "integration_seconds"))
    assert s <= report_value(text, "total_seconds") * 1.05 + 1e-9
    keys = [line.split(" = ")[0] for line in text.splitlines()]
    assert keys[:6] == ["method", "mesh", "sources", "vertices", "edges", "faces"]  # report.hpp:94-135 order


def test_threads_environment(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "square_env.obj", "unit_square")
    rep = str(tmp_path / "env.report")
    assert run(cli, ["distance", "--mesh", mesh, "--source", "0", "--report", rep],
               env={"GEOHEAT_THREADS": "3"}).returncode == 0
    assert report_value(open(rep).read(), "threads") == 3.0
    assert run(cli, ["distance", "--mesh", mesh, "--source", "0", "--threads", "2", "--report", rep],
               env={"GEOHEAT_THREADS": "3"}).returncode == 0
    assert report_value(open(rep).read(), "threads") == 2.0


def test_output_formats(gpu, ref, cli, tmp_path):
    mesh, P, F = write_mesh(gpu, ref, tmp_path, "square_fmt.obj", "unit_square")
    csv, ply, txt = (str(tmp_path / f"fmt.{x}") for x in ("csv", "ply", "txt"))
    for fmt, path in (("csv", csv), ("ply", ply), ("txt", txt)):
        r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--seq", "--out-format", fmt, "--out", path])
        assert r.returncode == 0, r.stderr
    lines = open(csv).read().splitlines()
    assert lines[0] == "vertex_index,distance" and len(lines) == 5
    expected = read_txt(txt)
    data = open(ply, "rb").read()
    head = data.index(b"end_header\n") + 11
    assert b"element vertex 4" in data[:head] and b"element face 2" in data[:head]
    rows = np.frombuffer(data[head:head + 32 * 4], dtype="<f8").reshape(4, 4)
    assert np.array_equal(rows[:, :3], P) and np.array_equal(rows[:, 3], expected)
    # stdout output is the same bytes as --out
    r = run(cli, ["distance", "--mesh", mesh, "--source", "0", "--seq"])
    assert r.stdout == open(txt, "rb").read()


def test_bench_csv_sweep(gpu, ref, cli, tmp_path):
    mesh, *_ = write_mesh(gpu, ref, tmp_path, "bench_sphere.obj", "icosphere", 2)
    r = run(cli, ["bench", "--mesh", mesh, "--methods", "face,edge", "--threads-list", "1,2", "--repeats", "2",
                  "--gs-iters", "60"])
    assert r.returncode == 0, r.stderr
    lines = r.stdout.decode().splitlines()
    assert lines[0].startswith("method,threads,repeat") and "distance_hash" in lines[0]
    rows = [line.split(",") for line in lines[1:]]
    assert len(rows) == 8 and all(len(c) >= 17 for c in rows)
    by = {}
    for c in rows:
        by.setdefault(c[0], set()).add((c[11], c[16]))
    assert all(len(v) == 1 for v in by.values())
    face_bytes = int(next(iter(by["face"]))[0])
    edge_bytes = int(next(iter(by["edge"]))[0])
    assert edge_bytes * 2 <= face_bytes  # the memory claim on a closed mesh


def test_subdivide(gpu, ref, cli, tmp_path):
    g = gpu.geoheat
    mesh, P, F = write_mesh(gpu, ref, tmp_path, "sub_square.obj", "unit_square")
    out1, out0 = str(tmp_path / "sub1.obj"), str(tmp_path / "sub0.obj")
    r = run(cli, ["subdivide", "--mesh", mesh, "--levels", "1", "--out", out1])
    assert r.returncode == 0 and b"vertices = 9" in r.stderr
    fine = g.load_mesh(out1)
    assert fine.vertex_count() == 9 and fine.face_count() == 8
    assert np.array_equal(fine.download("positions").reshape(-1, 3)[:4], P)
    assert run(cli, ["subdivide", "--mesh", mesh, "--levels", "0", "--out", out0]).returncode == 0
    same = g.load_mesh(out0)
    assert np.array_equal(same.download("positions").reshape(-1, 3), P)
    assert np.array_equal(same.download("faces").reshape(-1, 3), F)
    # byte-identical to the reference's subdivision + save_obj
    om = ref.subdivide(ref.build_mesh(P, F), 1)
    assert open(out1, "rb").read() == ref.save_mesh(om, 0)
    assert run(cli, ["subdivide", "--mesh", mesh, "--levels", "-1", "--out", out1]).returncode == 2


@pytest.mark.parametrize("method", ["face", "edge", "poisson"])
def test_cli_distances_match_reference_chain(gpu, ref, cli, tmp_path, method):
    """CLI output vs the reference's own chain on the same file: h, t and tau are
    the reference's left-to-right sums bit for bit, so face / edge output files
    are byte-identical to what the reference writes; CG (poisson) agrees to 1e-9."""
    mesh, P, F = write_mesh(gpu, ref, tmp_path, "torus.ply", "torus", 40, 20)
    out, rep = str(tmp_path / "d.txt"), str(tmp_path / "r.txt")
    r = run(cli, ["distance", "--mesh", mesh, "--source", "3,77", "--method", method, "--gs-iters", "300",
                  "--out", out, "--report", rep])
    assert r.returncode == 0, r.stderr
    om = ref.build_mesh(P, F)
    text = open(rep).read()
    assert report_value(text, "avg_edge_length") == om.average_edge_length()
    assert report_value(text, "t") == om.diffusion_time(1.0)
    assert report_value(text, "tau") == om.triangulation_quality()
    d = read_txt(out)
    if method == "poisson":
        d_ref, _, _ = ref.poisson(om, [3, 77], om.diffusion_time(1.0), 1e-5)
        np.testing.assert_allclose(d, d_ref, rtol=1e-9, atol=1e-12)
    else:
        from oracle.oracle import run_pipeline
        d_ref = run_pipeline(ref, P, F, [3, 77], sweeps=300, method=method)["d"]
        assert open(out, "rb").read() == ref.write_distances(d_ref, False)
