"""Parity of the B200 path with the reference (GPU, through the C ABI).

Bar: bit-identical per-element results (TriMesh arrays, BFS levels/parents/
rings, u, H, zero_count, G, X, distances) against the golden fixtures made by
the unmodified reference and against the C oracle on the same seeded inputs;
ADMM iteration counts and stop decisions identical, residual histories within
1e-12 relative (the device sums in a fixed tree order, the reference left to
right). Full-size configs are covered by reduced-sweep bitwise runs and by
size-independent properties (determinism, maximum principle, BFS invariants).
"""
import glob
import json
import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT
from oracle.oracle import ARRAYS

pytestmark = pytest.mark.gpu

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
INDEX = json.load(open(os.path.join(GOLDEN, "index.json")))
RESIDUAL_RTOL = 1e-12


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def assert_same(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    if not np.array_equal(bits(a.ravel()), bits(b.ravel())):
        diff = np.flatnonzero(bits(a.ravel()) != bits(b.ravel()))
        raise AssertionError(f"{what}: {diff.size} elements differ, first at {diff[:5]}")


def check_history(got, want, what):
    assert len(got) == len(want), what
    for g, w in zip(got, want):
        assert g == pytest.approx(w, rel=RESIDUAL_RTOL, abs=1e-300), what


@pytest.mark.parametrize("case", CASES)
def test_golden_case_bitwise(gpu, case):
    gh = gpu
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    mesh = gh.build_mesh(g["positions"], g["faces"])
    for name, _ in ARRAYS:
        assert_same(mesh.download(name).ravel(), g["mesh_" + name].ravel(), name)
    lv = gh.bfs_levels(mesh, g["sources"])
    assert_same(lv.level_of_vertex, g["level_of_vertex"], "level")
    assert_same(lv.parent_of_vertex, g["parent_of_vertex"], "parent")
    assert_same(lv.order, g["order"], "rings")
    assert_same(lv.offsets, g["offsets"], "ring offsets")
    assert lv.unreachable_count == int(g["unreachable"])
    t, sweeps, iters = float(g["t"]), int(g["sweeps"]), int(g["admm_iters"])
    assert gh.average_edge_length(mesh) == float(g["avg_edge_length"])  # left-to-right sum, bit for bit
    u = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps))
    assert_same(u, g["u"], "u")
    nh = gh.normalized_target_gradients(mesh, u)
    assert_same(nh.field, g["H"], "H")
    assert nh.zero_count == int(g["zero_count"])
    cfg = gh.AdmmConfig(max_iterations=iters)
    fr = gh.admm_face_optimize(mesh, g["H"], cfg)
    er = gh.admm_edge_optimize(mesh, g["H"], cfg)
    for tag, r, field, key in (("face", fr, fr.gradients, "G"), ("edge", er, er.differences, "X")):
        assert r.report.iterations == int(g[f"{tag}_iterations"]), tag
        assert r.report.converged == bool(g[f"{tag}_converged"]), tag
        check_history(r.report.primal_history, g[f"{tag}_primal"], tag + " primal")
        check_history(r.report.dual_history, g[f"{tag}_dual"], tag + " dual")
        assert r.report.state_bytes_formula == int(g[f"{tag}_state_bytes_formula"])
        assert_same(field, g[key], key)
    d_face = gh.integrate_face_gradients(mesh, lv, g["G"])
    d_edge = gh.integrate_edge_differences(mesh, lv, g["X"])
    assert_same(d_face, g["d_face"], "d_face")
    assert_same(d_edge, g["d_edge"], "d_edge")
    assert gh.field_hash(d_face) == int(g["hash_d_face"])
    if "u_warm3" in g:
        u2 = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=3), initial=u)
        assert_same(u2, g["u_warm3"], "warm start")
    e1 = gh.diffusion_residual(mesh, u, t, g["sources"], levels=lv)
    assert e1 == float(g["e1"])  # left-to-right sum, bit for bit
    # the fused device-resident chain equals the stage-by-stage results
    for method, key in (("face", "d_face"), ("edge", "d_edge")):
        d, rep = gh.distance(lv, method, sweeps, t, admm=cfg)
        assert_same(d, g[key], "fused " + method)
        assert rep.zero_count == int(g["zero_count"])


@pytest.mark.parametrize("name", sorted(INDEX["errors"]))
def test_mesh_errors_match_reference(gpu, name):
    e = INDEX["errors"][name]
    with pytest.raises(gpu.MeshError) as info:
        gpu.build_mesh(np.asarray(e["positions"], float), np.asarray(e["faces"], np.int32))
    assert str(info.value) == e["message"]


def test_invalid_arguments(gpu):
    gh = gpu
    g = np.load(os.path.join(GOLDEN, "unit_square.npz"))
    mesh = gh.build_mesh(g["positions"], g["faces"])
    with pytest.raises(ValueError, match="empty source set"):
        gh.bfs_levels(mesh, [])
    with pytest.raises(ValueError, match="out of range"):
        gh.bfs_levels(mesh, [9])
    lv = gh.bfs_levels(mesh, [0])
    with pytest.raises(ValueError, match="t must be positive"):
        gh.gs_diffuse(mesh, lv, 0.0, gh.DiffusionConfig(sweeps=1))
    with pytest.raises(ValueError, match="mu must be positive"):
        gh.admm_face_optimize(mesh, g["H"], gh.AdmmConfig(mu=0.0))
    with pytest.raises(ValueError, match="m must be positive"):
        gh.diffusion_time(mesh, -1.0)


def _oracle_chain(o, w, sweeps, t):
    mesh = o.build_mesh(w.positions, w.faces)
    lv = mesh.bfs(w.sources)
    if t is None:
        t = mesh.diffusion_time(w.m)
    u, _ = mesh.gs_diffuse(lv, t, sweeps)
    H, zc = mesh.normalized_target_gradients(u)
    G, fr = mesh.admm_face(H)
    X, er = mesh.admm_edge(H)
    return dict(t=t, level=lv.level_of_vertex, parent=lv.parent_of_vertex, u=u, H=H, zc=zc, G=G, X=X, fr=fr, er=er,
                d_face=mesh.integrate_face(lv, G), d_edge=mesh.integrate_edge(lv, X))


@pytest.mark.parametrize("config,scale,sweeps", [(2, 8, 400), (3, 16, 300), (4, 64, 200), (5, 128, 200)])
def test_configs_reduced_size_vs_oracle(gpu, port_oracle, config, scale, sweeps):
    """BASELINE configs 2-5 at reduced linear size, every stage bitwise vs the C oracle."""
    from paper_1812_06060_b200 import meshgen
    gh = gpu
    w = meshgen.config(config, scale=scale)
    ref = _oracle_chain(port_oracle, w, sweeps, w.t)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    assert_same(lv.level_of_vertex, ref["level"], "level")
    assert_same(lv.parent_of_vertex, ref["parent"], "parent")
    u = gh.gs_diffuse(mesh, lv, ref["t"], gh.DiffusionConfig(sweeps=sweeps))
    assert_same(u, ref["u"], "u")
    for method, key in (("face", "d_face"), ("edge", "d_edge")):
        d, rep = gh.distance(lv, method, sweeps, ref["t"])
        assert_same(d, ref[key], f"C{config} {method} distances")
        r = ref["fr"] if method == "face" else ref["er"]
        assert rep.admm_iterations == r.iterations and rep.converged == r.converged
        assert rep.zero_count == ref["zc"]


def test_config1_full_with_device_t(gpu, port_oracle):
    """Config 1 end to end with t from the device mean edge length: t is the
    reference's left-to-right sum bit for bit (gh_seqsum.cu), so the distances
    are bit-identical, and the error vs the great-circle geodesic equals the
    reference's."""
    from paper_1812_06060_b200 import meshgen
    gh = gpu
    w = meshgen.config(1)
    g = np.load(os.path.join(GOLDEN, "icosphere5_config1.npz"))
    d, rep = gh.distance_host(w.positions, w.faces, w.sources, "face", 1000, None, 1.0)
    assert np.float64(rep.t).view(np.uint64) == np.float64(g["t"]).view(np.uint64), (rep.t, float(g["t"]))
    assert_same(d, g["d_face"], "C1 distances with the device t")
    P = w.positions
    exact = np.arccos(np.clip(P @ P[0] / (np.linalg.norm(P, axis=1) * np.linalg.norm(P[0])), -1, 1))
    mask = np.arange(len(d)) != 0
    eps_gpu = np.sum(np.abs(d[mask] - exact[mask]) / exact[mask]) / len(d)
    eps_ref = np.sum(np.abs(g["d_face"][mask] - exact[mask]) / exact[mask]) / len(d)
    assert eps_gpu == pytest.approx(eps_ref, rel=1e-9)
    assert eps_ref == pytest.approx(0.047449, rel=1e-4)  # eps_face = 4.7449 %


@pytest.mark.slow
def test_config3_full_size_properties(gpu, port_oracle):
    """Config 3 at full size (8.4M vertices): mesh + BFS bitwise vs the oracle,
    3 sweeps bitwise, and the full 1000-sweep solve deterministic and inside
    the maximum-principle bound 0 <= u <= 1/min A_s (test_diffusion.cpp:92-109)."""
    from paper_1812_06060_b200 import meshgen
    gh = gpu
    w = meshgen.config(3)
    om = port_oracle.build_mesh(w.positions, w.faces)
    ol = om.bfs(w.sources)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    for name in ("edge_vertices", "vv_index", "vv_weight", "vertex_area", "vertex_weight_sum"):
        assert_same(mesh.download(name).ravel(), om.array(name), name)
    assert_same(lv.level_of_vertex, ol.level_of_vertex, "level")
    assert_same(lv.parent_of_vertex, ol.parent_of_vertex, "parent")
    t = om.diffusion_time(1.0)
    u3, _ = om.gs_diffuse(ol, t, 3)
    assert_same(gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=3)), u3, "u after 3 sweeps")
    a = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=1000))
    b = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=1000))
    assert_same(a, b, "determinism")
    va = om.array("vertex_area")
    assert a.min() >= 0.0 and a.max() <= 1.0 / va[w.sources].min() * (1 + 1e-12)


def test_cpp_wrapper_runs_reference_chain(gpu):
    """The C++ drop-in (include/geoheat_b200.hpp) reproduces the reference's config-1 hashes."""
    from paper_1812_06060_b200 import _build
    exe = os.path.join(_build.LIBDIR, "wrapper_parity")
    if not os.path.exists(exe):
        src = os.path.join(ROOT, "tests", "cpp", "wrapper_parity.cpp")
        _build.build_meshgen()
        subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"), src, "-o", exe, "-L",
                        _build.LIBDIR, "-lgeoheat_b200", "-lgh_meshgen", f"-Wl,-rpath,{_build.LIBDIR}"], check=True)
    t = float(np.load(os.path.join(GOLDEN, "icosphere5_config1.npz"))["t"])
    gpu.geoheat.release_cached_memory()
    r = subprocess.run([exe, t.hex()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout


TOL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "tol", "*.npz")))


@pytest.mark.parametrize("group", [None, "1", "3", "7"])
@pytest.mark.parametrize("case", TOL_CASES)
def test_residual_tolerance_early_stop(gpu, case, group, monkeypatch):
    """gs_diffuse with residual_tolerance (diffusion.hpp:110-117): same stop sweep, bitwise u,
    and the E1 history bit-identical (the reference's left-to-right sum of r^2 is
    reproduced exactly on the device). The sweeps run pipelined in groups whose
    every sweep is snapshot; GH_TOL_GROUP forces small groups so the stop falls
    inside, at the end of, and across groups."""
    if group:
        monkeypatch.setenv("GH_TOL_GROUP", group)
    gh = gpu
    g = np.load(os.path.join(GOLDEN, "tol", case + ".npz"))
    mesh = gh.build_mesh(g["positions"], g["faces"])
    lv = gh.bfs_levels(mesh, g["sources"])
    rep = gh.SolverReport()
    cfg = gh.DiffusionConfig(sweeps=int(g["sweeps"]), residual_tolerance=float(g["tolerance"]))
    u = gh.gs_diffuse(mesh, lv, float(g["t"]), cfg, rep)
    assert rep.iterations == int(g["iterations"]) and rep.converged == bool(g["converged"])
    assert_same(u, g["u"], "u")
    assert_same(np.asarray(rep.residual_history), g["residual_history"], "E1 history")


@pytest.mark.parametrize("nbands", [2, 3, 4, 8])
def test_band_sharded_diffusion_bitwise(gpu, nbands):
    """The multi-GPU band schedule (ghost levels written by the neighbour band
    through its peer pointers + per-level counters), emulated with all bands in
    one launch on this GPU: bit-identical to gs_diffuse on every fixture with
    enough levels and on config 3 at reduced size."""
    from paper_1812_06060_b200 import bands, meshgen
    gh = gpu
    for case in CASES:
        g = np.load(os.path.join(GOLDEN, case + ".npz"))
        if len(g["offsets"]) - 1 < nbands or int(g["sweeps"]) == 0:
            continue
        mesh = gh.build_mesh(g["positions"], g["faces"])
        lv = gh.bfs_levels(mesh, g["sources"])
        u = bands.gs_diffuse_bands(mesh, lv, nbands, float(g["t"]), int(g["sweeps"]))
        assert_same(u, g["u"], f"{case} with {nbands} bands")
    w = meshgen.config(3, scale=8)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    t = gh.diffusion_time(mesh, 1.0)
    one = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=200))
    assert_same(bands.gs_diffuse_bands(mesh, lv, nbands, t, 200), one, f"config 3/8 with {nbands} bands")


@pytest.mark.parametrize("nslices", [1, 2, 3, 5, 8])
def test_slice_sharded_diffusion_bitwise(gpu, port_oracle, nslices):
    """Sector slices (every slice owns 1/N of every ring; foreign neighbours are
    ghost rows their owners store into, counted per source slice and level),
    emulated with all slices in one launch on this GPU: bit-identical to the
    reference on every fixture (cold and warm start), on configs 2-5 at reduced
    size (config 4 in Morton ring order), and the ghost/export bookkeeping is
    consistent (every reachable vertex owned by exactly one slice)."""
    from paper_1812_06060_b200 import bands, meshgen
    gh = gpu
    for case in CASES:
        g = np.load(os.path.join(GOLDEN, case + ".npz"))
        if int(g["sweeps"]) == 0:
            continue
        mesh = gh.build_mesh(g["positions"], g["faces"])
        lv = gh.bfs_levels(mesh, g["sources"])
        u = bands.gs_diffuse_slices(mesh, lv, nslices, float(g["t"]), int(g["sweeps"]))
        assert_same(u, g["u"], f"{case} with {nslices} slices")
        if "u_warm3" in g.files:
            uw = bands.gs_diffuse_slices(mesh, lv, nslices, float(g["t"]), 3, initial=g["u"])
            assert_same(uw, g["u_warm3"], f"{case} warm start, {nslices} slices")
    for config, scale, sweeps in ((2, 8, 150), (3, 8, 200), (4, 64, 120), (5, 128, 100)):
        w = meshgen.config(config, scale=scale)
        om = port_oracle.build_mesh(w.positions, w.faces)
        ol = om.bfs(w.sources)
        t = om.diffusion_time(1.0) if w.t is None else w.t
        ref, _ = om.gs_diffuse(ol, t, sweeps)
        mesh = gh.build_mesh(w.positions, w.faces)
        lv = gh.bfs_levels(mesh, w.sources)
        assert_same(bands.gs_diffuse_slices(mesh, lv, nslices, t, sweeps), ref, f"C{config} {nslices} slices")
        if config == 3:
            owned = np.zeros(mesh.vertex_count(), np.int64)
            parts = [bands.Band(lv, r, nslices, partition="slices") for r in range(nslices)]
            for p in parts:
                owned += p.own_mask()
            reach = lv.level_of_vertex >= 0
            assert np.all(owned[reach] == 1) and np.all(owned[~reach] == 0)


def test_slice_blobs_connect_all(gpu):
    """Multi-process slice handles: every rank's IPC blob; connect_all refuses a
    blob list in the wrong order or from another partition before mapping."""
    from paper_1812_06060_b200 import bands
    gh = gpu
    g = np.load(os.path.join(GOLDEN, "icosphere3.npz"))
    mesh = gh.build_mesh(g["positions"], g["faces"])
    lv = gh.bfs_levels(mesh, g["sources"])
    parts = [bands.Band(lv, r, 3, partition="slices") for r in range(3)]
    blobs = [p.export() for p in parts]
    with pytest.raises(ValueError, match="not slice"):
        parts[0].connect_all([blobs[0], blobs[2], blobs[1]])
    other = bands.Band(lv, 1, 2, partition="slices").export()
    with pytest.raises(ValueError, match="not slice"):
        parts[0].connect_all([blobs[0], other, blobs[2]])
    with pytest.raises(ValueError, match="gh_band_connect_all"):
        parts[0].connect(None, blobs[1])


def test_band_export_and_neighbour_checks(gpu):
    """Multi-process band handles: the IPC blob round-trips and connect() refuses
    a blob that is not the adjacent band (before any peer mapping)."""
    from paper_1812_06060_b200 import bands
    gh = gpu
    g = np.load(os.path.join(GOLDEN, "icosphere3.npz"))
    mesh = gh.build_mesh(g["positions"], g["faces"])
    lv = gh.bfs_levels(mesh, g["sources"])
    b0, b1, b2 = (bands.Band(lv, r, 3) for r in range(3))
    plan = bands.plan_bands(lv.offsets, 3)
    assert [b0.lb, b0.le, b1.lb, b1.le, b2.lb, b2.le] == [plan[0], plan[1], plan[1], plan[2], plan[2], plan[3]]
    blobs = [b.export() for b in (b0, b1, b2)]
    assert len(set(map(len, blobs))) == 1
    with pytest.raises(ValueError, match="lower neighbour"):
        b2.connect(blobs[0], None)  # band 0 is not band 2's lower neighbour
    with pytest.raises(ValueError, match="upper neighbour"):
        b0.connect(None, blobs[2])


def test_dropin_reference_program_bitwise(gpu):
    """tests/cpp/dropin_run_pipeline.cpp: the same run_pipeline chain compiled with
    the reference's functions and with geoheat::b200 on the reference's own types;
    built in the build container (needs /root/reference), run here."""
    from paper_1812_06060_b200 import _build
    exe = os.path.join(_build.LIBDIR, "dropin_run_pipeline")
    if not os.path.exists(exe):
        pytest.skip("drop-in program not prebuilt (built by tests/test_abi.py in the build container)")
    gpu.geoheat.release_cached_memory()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("identical") == 6, r.stdout


def _fan(n):
    """A two-ring disc around one hub vertex of valence n (past 16 bits for
    n > 65535): hub 0, inner ring 1..n, outer ring n+1..2n."""
    a = np.arange(n)
    th = 2 * np.pi * a / n
    inner = np.stack([np.cos(th), np.sin(th), 0.1 * np.sin(3 * th)], 1)
    outer = np.stack([2 * np.cos(th + np.pi / n), 2 * np.sin(th + np.pi / n), np.zeros(n)], 1)
    P = np.concatenate([[[0.0, 0.0, 0.3]], inner, outer])
    i0, i1 = 1 + a, 1 + (a + 1) % n
    o0, o1 = 1 + n + a, 1 + n + (a + 1) % n
    F = np.concatenate([np.stack([np.zeros(n, np.int64), i0, i1], 1), np.stack([i0, o0, i1], 1),
                        np.stack([i1, o0, o1], 1)]).astype(np.int32)
    return P, F


@pytest.mark.parametrize("n,source", [(70_000, "outer"), (70_000, "hub"), (65_535, "outer"), (131_072, "inner")])
def test_high_valence_hub_bitwise(gpu, port_oracle, n, source):
    """A vertex whose valence does not fit the 16-bit row length of the
    diffusion layout (deg_big path): every stage bitwise vs the C oracle, one
    launch and band-sharded."""
    from types import SimpleNamespace
    from paper_1812_06060_b200 import bands
    gh = gpu
    P, F = _fan(n)
    src = np.array([{"outer": n + 1, "hub": 0, "inner": 1}[source]], np.int32)
    w = SimpleNamespace(positions=P, faces=F, sources=src, m=1.0)
    ref = _oracle_chain(port_oracle, w, 60, None)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, src)
    assert_same(lv.level_of_vertex, ref["level"], "level")
    u = gh.gs_diffuse(mesh, lv, ref["t"], gh.DiffusionConfig(sweeps=60))
    assert_same(u, ref["u"], "u")
    for method, key in (("face", "d_face"), ("edge", "d_edge")):
        d, rep = gh.distance(lv, method, 60, ref["t"])
        assert_same(d, ref[key], f"fan {n} {method} distances")
    if len(lv.offsets) - 1 >= 2:
        assert_same(bands.gs_diffuse_bands(mesh, lv, 2, ref["t"], 60), ref["u"], "fan with 2 bands")


@pytest.mark.parametrize("mode", ["auto", "col32", "win2", "win3", "win2_mixed", "win3_mixed", "morton",
                                  "morton_win3_mixed", "morton_col32", "group1", "group7", "group16_normal",
                                  "group3_period", "general", "general_win3"])
def test_diffusion_column_formats_bitwise(gpu, port_oracle, monkeypatch, mode):
    """The diffusion kernel streams 16-bit column offsets into 2 or 3 per-chunk
    windows (chunks whose windows do not fit keep 32-bit columns and take the
    global-memory path); every format, and mixes forced by a tiny window
    limit, give u bit-identical to the reference on every fixture and on
    reduced configs 2-5, single band and 3 bands. The "morton" modes lay each
    ring out in spatial order (the layout picked when vertex-id order leaves no
    16-bit format usable), which moves rows between chunks but not their sums.
    The "group" modes run the sweeps in groups of K (one pipeline per group,
    DESIGN.md §3.4): the same tasks in another order, so the same bits. The
    "general" modes run the single band through the instances that decide
    snapshots and neighbour copies at run time (the plain solve takes lean ones)."""
    from paper_1812_06060_b200 import bands, meshgen
    gh = gpu
    if mode.startswith("general"):
        monkeypatch.setenv("GH_DIFFUSE_GENERAL", "1")
        mode = mode[8:] or "auto"
    if mode.startswith("group"):  # sweep groups (GH_SWEEP_GROUP): same tasks, another step order
        k = mode[5:].split("_")[0]
        monkeypatch.setenv("GH_SWEEP_GROUP", k)
        if mode.endswith("normal"):
            monkeypatch.setenv("GH_STREAM_L2", "2")
        if mode.endswith("period"):
            monkeypatch.setenv("GH_SWEEP_PERIOD", "5000")
        mode = "auto"
    if mode.startswith("morton"):
        monkeypatch.setenv("GH_LAYOUT", "morton")
        mode = mode[7:] or "auto"
    if mode == "col32":
        monkeypatch.setenv("GH_DIFFUSE_COL32", "1")
    if mode.startswith("win"):
        monkeypatch.setenv("GH_COL16_WINDOWS", mode[3])
    if mode.endswith("mixed"):
        monkeypatch.setenv("GH_COL16_SPAN", "96")
    want_bits = 32 if mode == "col32" else 16
    for case in CASES:
        g = np.load(os.path.join(GOLDEN, case + ".npz"))
        if int(g["sweeps"]) == 0:
            continue
        mesh = gh.build_mesh(g["positions"], g["faces"])
        lv = gh.bfs_levels(mesh, g["sources"])
        u = gh.gs_diffuse(mesh, lv, float(g["t"]), gh.DiffusionConfig(sweeps=int(g["sweeps"])))
        assert_same(u, g["u"], f"{case} ({mode})")
        if lv.unreachable_count < mesh.vertex_count():
            assert lv.column_bits == want_bits, case
    for config, scale, sweeps in ((2, 8, 300), (3, 16, 300), (4, 64, 200), (5, 128, 100)):
        w = meshgen.config(config, scale=scale)
        om = port_oracle.build_mesh(w.positions, w.faces)
        ol = om.bfs(w.sources)
        t = om.diffusion_time(1.0) if w.t is None else w.t
        ref, _ = om.gs_diffuse(ol, t, sweeps)
        mesh = gh.build_mesh(w.positions, w.faces)
        lv = gh.bfs_levels(mesh, w.sources)
        assert_same(gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps)), ref, f"C{config} ({mode})")
        assert lv.column_bits == want_bits
        assert_same(bands.gs_diffuse_bands(mesh, lv, 3, t, sweeps), ref, f"C{config} 3 bands ({mode})")


def test_repeated_solves_reuse_cached_blocks(gpu):
    """Device blocks are recycled by exact size across solves (gh_alloc.cu):
    end-to-end solves of two meshes, interleaved and repeated (handles created
    and destroyed every time, so every large block comes from the cache after
    the first round), return the first round's distances bit for bit."""
    from paper_1812_06060_b200 import meshgen
    gh = gpu
    ws = [meshgen.config(2, scale=8), meshgen.config(3, scale=16)]
    first = []
    for rnd in range(3):
        for k, w in enumerate(ws):
            d, rep = gh.distance_host(w.positions, w.faces, w.sources, w.method, 200, w.t, w.m)
            if rnd == 0:
                first.append(d)
            else:
                assert_same(d, first[k], f"round {rnd}, mesh {k}")


def test_release_cached_memory_keeps_handles(gpu):
    """gh_release_cached_memory hands cached blocks back to the driver between
    solves: live handles keep working and results keep their bits."""
    from paper_1812_06060_b200 import meshgen
    gh = gpu
    w = meshgen.config(3, scale=16)
    mesh = gh.build_mesh(w.positions, w.faces)
    lv = gh.bfs_levels(mesh, w.sources)
    t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
    u1 = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=50))
    d1, _ = gh.distance(lv, "face", 50, t)
    gh.geoheat.release_cached_memory()
    u2 = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=50))
    gh.geoheat.release_cached_memory()
    d2, _ = gh.distance(lv, "face", 50, t)
    assert_same(u2, u1, "u after a release")
    assert_same(d2, d1, "distances after a release")


def _strip(nx: int, wobble: float = 0.013):
    """A 2 x nx triangle strip (a ladder): a source at one end gives ~nx BFS rings."""
    i = np.arange(nx, dtype=np.float64)
    P = np.zeros((2 * nx, 3))
    P[0::2, 0] = i
    P[1::2, 0] = i + 0.5 * np.sin(i)  # irregular cotan weights
    P[1::2, 1] = 1.0
    P[:, 2] = wobble * np.cos(0.7 * np.arange(2 * nx))
    a = 2 * np.arange(nx - 1, dtype=np.int32)
    F = np.concatenate([np.stack([a, a + 2, a + 3], 1), np.stack([a, a + 3, a + 1], 1)]).astype(np.int32)
    return P, F


@pytest.mark.parametrize("nbands", [1, 3])
def test_more_levels_than_the_shared_table(gpu, port_oracle, nbands):
    """More than 12,288 BFS rings (gh_diffuse.cu kMaxSmemLevels): the level table
    stays in global memory (k_diffuse_tma<*, false, *>); u bitwise vs the oracle,
    single band and the 3-band emulation, and the chain's distances bitwise."""
    gh = gpu
    from paper_1812_06060_b200 import bands as GB
    P, F = _strip(13_000)
    src = np.array([0], np.int32)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, src)
    assert lv.level_count() > 12 * 1024
    om = port_oracle.build_mesh(P, F)
    ol = om.bfs(src)
    assert_same(lv.level_of_vertex, ol.level_of_vertex, "level")
    t = om.diffusion_time(1.0)
    for sweeps in (1, 2, 37):
        want, _ = om.gs_diffuse(ol, t, sweeps)
        if nbands == 1:
            got = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps))
        else:
            got = GB.gs_diffuse_bands(mesh, lv, nbands, t, sweeps)
        assert_same(got, want, f"u after {sweeps} sweeps, {nbands} band(s)")
    if nbands == 1:
        u, _ = om.gs_diffuse(ol, t, 37)
        H, _ = om.normalized_target_gradients(u)
        X, _ = om.admm_edge(H, 10)
        d, _ = gh.distance(lv, "edge", 37, t)
        assert_same(d, om.integrate_edge(ol, X), "edge-method distances")


def test_pageable_and_pinned_uploads_agree(gpu):
    """Large pageable host arrays go through pinned staging slots filled by host
    threads (both ways: mesh upload, result download); sizes past the staging
    threshold and not a multiple of the 16 MiB slot must give the same bits as
    the pinned path (the driver's async copies)."""
    import ctypes as C
    from paper_1812_06060_b200 import geoheat as G, meshgen
    gh = gpu
    P, F, S = meshgen.torus(2900, 1500, 1.0, 0.3, 3e-4, 4, 2)  # 104 MB positions and faces, 35 MB distances
    Fi = np.ascontiguousarray(F, np.int32)
    n = P.shape[0]
    assert P.nbytes % (16 << 20) and 8 * n > (32 << 20)
    L = G._lib.load()
    mesh_a = gh.build_mesh(P, Fi)  # pageable -> staged
    pp, pf, pd = C.c_void_p(), C.c_void_p(), C.c_void_p()
    for ptr, nb in ((pp, P.nbytes), (pf, Fi.nbytes), (pd, 8 * n)):
        G._check(L.gh_host_alloc(nb, C.byref(ptr)))
    try:
        C.memmove(pp, P.ctypes.data, P.nbytes)
        C.memmove(pf, Fi.ctypes.data, Fi.nbytes)
        h = C.c_void_p()
        G._check(L.gh_mesh_create(pp, n, pf, Fi.shape[0], C.byref(h)))
        mesh_b = G.TriMesh(h)  # pinned -> async copies
        for name in ("positions", "faces", "vv_weight", "vertex_area", "face_area", "vv_index"):
            assert np.array_equal(mesh_a.download(name).view(np.uint8), mesh_b.download(name).view(np.uint8)), name
        del mesh_b
        # the result into pageable memory (staged) and into pinned memory (async copy)
        d_page, _ = gh.distance_host(P, Fi, S, "face", 20, None, 1.0)
        Sa = np.ascontiguousarray(S, np.int32)
        pcfg = G._pipeline_config("face", 20, None, 1.0, G.AdmmConfig())
        rr = G.gh_run_report()
        G._check(L.gh_distance_host(pp, n, pf, Fi.shape[0], Sa.ctypes.data_as(C.c_void_p), Sa.size, C.byref(pcfg), pd,
                                    C.byref(rr)))
        d_pin = np.ctypeslib.as_array(C.cast(pd, C.POINTER(C.c_double)), shape=(n,)).copy()
        assert np.array_equal(d_page.view(np.uint64), d_pin.view(np.uint64))
    finally:
        for ptr in (pp, pf, pd):
            L.gh_host_free(ptr)


def _ribbon(nx: int, ny: int, seed: int = 5):
    """A jittered ny-wide, nx-long triangulated ribbon: a corner source gives ~nx + ny BFS rings of <= ny + 1 vertices."""
    rng = np.random.default_rng(seed)
    x, y = np.meshgrid(np.arange(nx, dtype=np.float64), np.arange(ny, dtype=np.float64), indexing="ij")
    P = np.stack([x, y, 0.05 * np.sin(0.3 * x) * np.cos(0.4 * y)], -1).reshape(-1, 3)
    P[:, :2] += rng.uniform(-0.2, 0.2, (nx * ny, 2))
    i, j = np.meshgrid(np.arange(nx - 1), np.arange(ny - 1), indexing="ij")
    a = (i * ny + j).ravel()
    b, c, d = a + ny, a + ny + 1, a + 1
    flip = ((i + j) & 1).ravel().astype(bool)
    F = np.where(flip[:, None, None], np.stack([np.stack([a, b, d], 1), np.stack([b, c, d], 1)], 1),
                 np.stack([np.stack([a, b, c], 1), np.stack([a, c, d], 1)], 1)).reshape(-1, 3).astype(np.int32)
    return P, F


@pytest.mark.parametrize("m,expect", [(1.0, "truncated"), (40.0, "widened"), (1.0, "partial")])
def test_zero_level_truncation_bitwise(zero_skipping, port_oracle, m, expect, monkeypatch):
    """gs_diffuse on a mesh with far more rings than the heat reaches: only the
    levels below a verified cap are updated, in several launches. u is the oracle's bit for
    bit, equal to the plain launch's (truncation off), for sweep counts that end inside the
    first, a middle and the last launch. "widened": a first cap of 128 levels and a margin of
    8 (the heat reaches ~500 rings in one sweep and ~640 by sweep 71), so the first launch and
    later ones are undone and redone with larger caps."""
    gh = zero_skipping
    if expect == "widened":
        monkeypatch.setenv("GH_ZERO_LEVELS_FIRST", "128")
        monkeypatch.setenv("GH_ZERO_LEVELS_MARGIN", "8")
    if expect == "partial":
        # the diffusion layout covers the first 600 rings only (bfs_build lays out 2048 on large
        # meshes); the second launch's cap (front ~476 + 161) passes it, so the band is rebuilt with
        # more levels and the state carried over; the plain launches rebuild it over every level
        monkeypatch.setenv("GH_PARTIAL_LEVELS", "600")
        monkeypatch.setenv("GH_ZERO_LEVELS_FIRST", "512")
    P, F = _ribbon(3000, 12)
    src = np.array([0], np.int32)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, src)
    reach = P.shape[0]
    assert lv.level_count() > 2500
    om = port_oracle.build_mesh(P, F)
    ol = om.bfs(src)
    t = om.diffusion_time(m)
    seen_retry = False
    assert lv.layout_levels == (600 if expect == "partial" else lv.level_count())
    for sweeps in (2, 3, 16, 71):
        want, _ = om.gs_diffuse(ol, t, sweeps)
        if expect == "partial":
            lv = gh.bfs_levels(mesh, src)  # a fresh partial layout (the plain launch below completes it)
        got = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps))
        st = lv.diffusion_stats
        if expect == "partial":
            assert lv.layout_levels == (600 if sweeps == 2 else 1200), (sweeps, lv.layout_levels)
        assert_same(got, want, f"u after {sweeps} sweeps (m = {m}), {st}")
        gh.set_zero_level_truncation(False)
        try:
            plain = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps))
            sp = lv.diffusion_stats
        finally:
            gh.set_zero_level_truncation(True)
        assert_same(plain, want, f"plain launch, {sweeps} sweeps")
        assert lv.layout_levels == lv.level_count()
        assert sp == {"active_levels": lv.level_count(), "launches": 1, "retries": 0, "row_updates": reach * sweeps}
        seen_retry |= st["retries"] > 0
        if expect in ("truncated", "partial"):
            assert st["retries"] == 0 and st["active_levels"] < lv.level_count(), st
            assert st["row_updates"] < reach * sweeps // 2, st
            assert st["launches"] == {2: 1, 3: 2, 16: 2, 71: 3}[sweeps], st
            # every value past the last launch's cap is +0
            far = lv.level_of_vertex >= st["active_levels"]
            assert far.any() and not got.view(np.uint64)[far].any()
        else:
            assert st["retries"] >= 2, st  # 128 -> 256 -> 512 in the first launch alone
    if expect == "widened":
        assert seen_retry
    if expect == "widened":
        # caps that keep failing until most of the mesh is inside: the solve goes back to every level
        # (900 rings, first cap 128: 128 and 256 are flagged, 512 holds more than half the vertices)
        P2, F2 = _ribbon(900, 12)
        mesh2 = gh.build_mesh(P2, F2)
        lv2 = gh.bfs_levels(mesh2, src)
        om2 = port_oracle.build_mesh(P2, F2)
        ol2 = om2.bfs(src)
        t2 = om2.diffusion_time(m)
        for sweeps in (2, 9):
            want2, _ = om2.gs_diffuse(ol2, t2, sweeps)
            assert_same(gh.gs_diffuse(mesh2, lv2, t2, gh.DiffusionConfig(sweeps=sweeps)), want2, "back to every level")
            st = lv2.diffusion_stats
            assert st["retries"] == 2 and st["active_levels"] == lv2.level_count() and st["launches"] == 3, st
    # the chain behind it (the ADMM skips the faces and edges that stay +0, gh_grad.cu): the
    # oracle's distances bit for bit, with and without the zero skipping, both methods
    u16, _ = om.gs_diffuse(ol, t, 16)
    H16, _ = om.normalized_target_gradients(u16)
    for method in ("face", "edge"):
        if method == "face":
            Gf, orep = om.admm_face(H16, 10)
            want_d = om.integrate_face(ol, Gf)
        else:
            Xe, orep = om.admm_edge(H16, 10)
            want_d = om.integrate_edge(ol, Xe)
        d1, r1 = gh.distance(lv, method, 16, t)
        gh.set_zero_level_truncation(False)
        try:
            d0, r0 = gh.distance(lv, method, 16, t)
        finally:
            gh.set_zero_level_truncation(True)
        assert_same(d1, want_d, f"{method} distances with zero skipping")
        assert_same(d0, want_d, f"{method} distances without zero skipping")
        assert r1.admm_iterations == r0.admm_iterations == orep.iterations and r1.converged == r0.converged
        assert np.float64(r1.final_primal).view(np.uint64) == np.float64(r0.final_primal).view(np.uint64)
        assert np.float64(r1.final_dual).view(np.uint64) == np.float64(r0.final_dual).view(np.uint64)
    # a warm start may be nonzero anywhere: the plain launch
    u1 = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=4), initial=want)
    assert lv.diffusion_stats["launches"] == 1 and lv.diffusion_stats["active_levels"] == lv.level_count()
    w1, _ = om.gs_diffuse(ol, t, 4, initial=want)
    assert_same(u1, w1, "warm start")


def test_zero_skipping_with_several_sources_and_an_unreachable_part(zero_skipping, port_oracle):
    """The exact-zero skipping (truncated diffusion, ADMM active sets, partial layout) on a long
    ribbon with sources at both ends and in the middle plus a second, unreachable ribbon: u and the
    distances of both methods are the oracle's bit for bit (unreachable vertices: u = 0, d = inf)."""
    gh = zero_skipping
    P1, F1 = _ribbon(9000, 10, seed=11)
    P2, F2 = _ribbon(300, 10, seed=12)
    P2 = P2 + np.array([0.0, 50.0, 0.0])
    P = np.concatenate([P1, P2])
    F = np.concatenate([F1, F2 + P1.shape[0]]).astype(np.int32)
    n1 = P1.shape[0]
    src = np.array([0, n1 - 1, (4500 * 10) + 5], np.int32)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, src)
    assert lv.unreachable_count == P2.shape[0] and lv.level_count() > 1024
    assert lv.layout_levels == lv.level_count()  # ~2250 rings from three sources, most vertices within 2048: every level laid out
    om = port_oracle.build_mesh(P, F)
    ol = om.bfs(src)
    t = om.diffusion_time(1.0)
    want, _ = om.gs_diffuse(ol, t, 40)
    got = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=40))
    st = lv.diffusion_stats
    assert_same(got, want, f"u, {st}")
    assert st["launches"] == 3 and st["active_levels"] < lv.level_count() and st["retries"] == 0, st
    H, _ = om.normalized_target_gradients(want)
    Gf, _ = om.admm_face(H, 10)
    Xe, _ = om.admm_edge(H, 10)
    d_face, _ = gh.distance(lv, "face", 40, t)
    d_edge, _ = gh.distance(lv, "edge", 40, t)
    assert_same(d_face, om.integrate_face(ol, Gf), "face distances")
    assert_same(d_edge, om.integrate_edge(ol, Xe), "edge distances")
    assert np.isinf(d_face[n1:]).all() and np.isfinite(d_face[:n1]).all()
