"""The CPU oracle, pinned before it is trusted (CPU only).

1. The C restatement (oracle/geoheat_oracle.c, `port`) reproduces every stage of
   the golden fixtures bit for bit. The fixtures were produced by the
   unmodified reference headers (tests/golden/make_golden.py).
2. Known-answer values restated from the reference's own unit tests
   (proj/tests/test_mesh.cpp, test_diffusion.cpp, test_integrate.cpp).
3. Where /root/reference exists (the build container), the port is also run
   side by side with the reference library on fresh seeded meshes.
"""
import glob
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN
from oracle.oracle import ARRAYS, Oracle, OracleMeshError, available

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))
INDEX = json.load(open(os.path.join(GOLDEN, "index.json")))


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.uint64) if a.dtype == np.float64 else a


def assert_same(a, b, what=""):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (what, a.shape, b.shape)
    assert np.array_equal(bits(a.ravel()), bits(b.ravel())), what


def run_port(o, g):
    mesh = o.build_mesh(g["positions"], g["faces"])
    lv = mesh.bfs(g["sources"])
    t = float(g["t"])
    u, _ = mesh.gs_diffuse(lv, t, int(g["sweeps"]))
    H, zc = mesh.normalized_target_gradients(u)
    G, fr = mesh.admm_face(H, int(g["admm_iters"]))
    X, er = mesh.admm_edge(H, int(g["admm_iters"]))
    return mesh, lv, u, H, zc, G, fr, X, er


@pytest.mark.parametrize("case", CASES)
def test_port_matches_reference_fixture(port_oracle, case):
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    mesh, lv, u, H, zc, G, fr, X, er = run_port(port_oracle, g)
    for name, _ in ARRAYS:
        assert_same(mesh.array(name), g["mesh_" + name], name)
    assert mesh.average_edge_length() == float(g["avg_edge_length"])
    assert_same(lv.level_of_vertex, g["level_of_vertex"], "level")
    assert_same(lv.parent_of_vertex, g["parent_of_vertex"], "parent")
    assert_same(lv.order, g["order"], "rings")
    assert_same(lv.offsets, g["offsets"], "ring offsets")
    assert lv.unreachable == int(g["unreachable"])
    assert_same(u, g["u"], "u")
    assert_same(H, g["H"], "H")
    assert zc == int(g["zero_count"])
    assert_same(G, g["G"], "G")
    assert_same(X, g["X"], "X")
    for tag, r in (("face", fr), ("edge", er)):
        assert r.iterations == int(g[f"{tag}_iterations"])
        assert r.converged == bool(g[f"{tag}_converged"])
        assert_same(r.primal_history, g[f"{tag}_primal"], tag + " primal")
        assert_same(r.dual_history, g[f"{tag}_dual"], tag + " dual")
        assert r.state_bytes_formula == int(g[f"{tag}_state_bytes_formula"])
    assert_same(mesh.integrate_face(lv, G), g["d_face"], "d_face")
    assert_same(mesh.integrate_edge(lv, X), g["d_edge"], "d_edge")
    assert port_oracle.field_hash(g["d_face"]) == int(g["hash_d_face"])
    if "u_warm3" in g:
        u2, _ = mesh.gs_diffuse(lv, float(g["t"]), 3, initial=u)
        assert_same(u2, g["u_warm3"], "warm start")
    assert mesh.diffusion_residual(u, float(g["t"]), g["sources"]) == float(g["e1"])


def test_config1_hashes_match_survey(port_oracle):
    # shim-built reference, icosphere_mesh(5), source 0, m = 1
    assert INDEX["cases"]["icosphere5_config1"]["hash_d_face"] == "cca540701b66bfd5"
    assert INDEX["cases"]["icosphere5_config1"]["hash_d_edge"] == "a8e56e8b98582eb9"
    assert INDEX["cases"]["icosphere5_config1"]["zero_count"] == 5560


@pytest.mark.parametrize("name", sorted(INDEX["errors"]))
def test_port_rejects_like_reference(port_oracle, name):
    e = INDEX["errors"][name]
    with pytest.raises(OracleMeshError) as info:
        port_oracle.build_mesh(np.asarray(e["positions"], float), np.asarray(e["faces"], np.int32))
    assert str(info.value) == e["message"]


def test_invalid_sources(port_oracle):
    g = np.load(os.path.join(GOLDEN, "unit_square.npz"))
    mesh = port_oracle.build_mesh(g["positions"], g["faces"])
    with pytest.raises(ValueError):
        mesh.bfs([])
    with pytest.raises(ValueError):
        mesh.bfs([9])


# ---- known answers restated from the reference's unit tests
def square(o):
    g = np.load(os.path.join(GOLDEN, "unit_square.npz"))
    return o.build_mesh(g["positions"], g["faces"])


def test_unit_square_known_answers(port_oracle):
    m = square(port_oracle)
    assert (m.nv, m.ne, m.nf, m.ni) == (4, 5, 2, 1)  # test_mesh.cpp:26-36
    assert np.allclose(m.array("face_area"), 0.5)
    va = m.array("vertex_area")
    assert va[1] == pytest.approx(1 / 6) and va[3] == pytest.approx(1 / 6)  # test_mesh.cpp:38-46
    assert va[0] == pytest.approx(1 / 3) and va[2] == pytest.approx(1 / 3)
    ev = m.array("edge_vertices").reshape(-1, 2)
    w = m.array("edge_weight")
    e01 = [i for i, (a, b) in enumerate(ev) if (a, b) == (0, 1)][0]
    e02 = [i for i, (a, b) in enumerate(ev) if (a, b) == (0, 2)][0]
    assert w[e01] == pytest.approx(0.5) and abs(w[e02]) <= 1e-15  # test_mesh.cpp:77-83
    assert m.average_edge_length() == pytest.approx((4 + math.sqrt(2)) / 5)  # test_mesh.cpp:214-217
    assert m.diffusion_time(1.0) == pytest.approx(1.17254, rel=1e-5)  # test_diffusion.cpp:18-22
    lv = m.bfs([0])
    assert lv.nlev == 2 and list(lv.order) == [0, 1, 2, 3]  # test_mesh.cpp:143-155
    assert list(lv.parent_of_vertex[1:]) == [0, 0, 0]


def test_square_diffusion_known_answers(port_oracle):
    m = square(port_oracle)
    lv = m.bfs([0])
    u, _ = m.gs_diffuse(lv, 1.0, 0)
    assert list(u) == [1.0, 0.0, 0.0, 0.0]  # test_diffusion.cpp:37-42
    u, _ = m.gs_diffuse(lv, 1.0, 1)
    va, ws = m.array("vertex_area"), m.array("vertex_weight_sum")
    assert u[0] == pytest.approx(1.0 / (va[0] + 1.0 * ws[0]))  # test_diffusion.cpp:43-49
    # 200 sweeps reach the dense solve of (A - t Lc) u = u0 (test_diffusion.cpp:50-56)
    off, idx, w = m.array("vv_offset"), m.array("vv_index"), m.array("vv_weight")
    A = np.diag(va + ws)
    for j in range(4):
        for a in range(off[j], off[j + 1]):
            A[j, idx[a]] -= w[a]
    exact = np.linalg.solve(A, np.array([1.0, 0, 0, 0]))
    u, _ = m.gs_diffuse(lv, 1.0, 200)
    assert np.allclose(u, exact, rtol=1e-8)
    assert m.diffusion_residual(exact, 1.0, [0]) <= 1e-12  # test_diffusion.cpp:113-116


def test_face_gradient_linear(port_oracle):
    m = square(port_oracle)
    P = m.array("positions").reshape(-1, 3)
    g = m.face_gradient(2 * P[:, 0] + 3 * P[:, 1])  # test_mesh.cpp:110-115
    assert np.abs(g - [2, 3, 0]).max() < 1e-13
    H, zc = m.normalized_target_gradients(2 * P[:, 0])  # test_diffusion.cpp:156-164
    assert zc == 0 and np.abs(H - [-1, 0, 0]).max() < 1e-14
    H, zc = m.normalized_target_gradients(np.full(4, 0.7))  # test_diffusion.cpp:165-171
    assert zc == 2 and not H.any()


def test_integrate_constant_field(port_oracle):
    m = square(port_oracle)
    lv = m.bfs([0])
    d = m.integrate_face(lv, np.array([[1.0, 0, 0], [1.0, 0, 0]]))  # test_integrate.cpp:14-24
    assert d[0] == 0 and d[1] == pytest.approx(1) and d[2] == pytest.approx(1) and abs(d[3]) <= 1e-15


def test_unreachable_is_infinite(port_oracle):
    g = np.load(os.path.join(GOLDEN, "two_disjoint_triangles.npz"))
    assert np.isinf(g["d_face"][3:]).all() and np.isfinite(g["d_face"][:3]).all()  # test_integrate.cpp:63-74


def test_state_bytes_formula(port_oracle):
    g = np.load(os.path.join(GOLDEN, "icosphere3.npz"))
    F, E = g["faces"].shape[0], g["mesh_edge_vertices"].size // 2
    assert int(g["face_state_bytes_formula"]) == (6 * F + 15 * E) * 8  # closed mesh: E_int = E
    assert int(g["edge_state_bytes_formula"]) == (6 * F + 2 * E) * 8 + 3 * F


# ---- live side by side with the reference (build container only)
@pytest.mark.skipif(not available("reference") or not os.path.isdir("/root/reference"),
                    reason="reference library needs /root/reference (build container)")
@pytest.mark.parametrize("seed", [1, 2])
def test_port_matches_reference_live(port_oracle, seed):
    from paper_1812_06060_b200 import meshgen
    ref = Oracle("reference")
    P, F, S = meshgen.torus(40 + 4 * seed, 22, 1.0, 0.3, 1e-3 * 0.3, seed, 3)
    out = []
    for o in (ref, port_oracle):
        mesh = o.build_mesh(P, F)
        lv = mesh.bfs(S)
        t = mesh.diffusion_time(1.0)
        u, _ = mesh.gs_diffuse(lv, t, 150)
        H, zc = mesh.normalized_target_gradients(u)
        G, fr = mesh.admm_face(H)
        X, er = mesh.admm_edge(H)
        out.append((u, H, G, X, mesh.integrate_face(lv, G), mesh.integrate_edge(lv, X), fr.primal_history,
                    er.dual_history))
    for a, b in zip(*out):
        assert_same(a, b)


@pytest.mark.skipif(not available("reference") or not os.path.isdir("/root/reference"),
                    reason="reference library needs /root/reference (build container)")
def test_threads_do_not_change_bits(port_oracle):
    # test_diffusion.cpp:75-90: results are bitwise thread-count invariant
    g = np.load(os.path.join(GOLDEN, "hex_disk12_two_sources.npz"))
    ref = Oracle("reference")
    outs = []
    for o in (ref, port_oracle):
        for th in (1, 4):
            o.set_threads(th)
            mesh = o.build_mesh(g["positions"], g["faces"])
            lv = mesh.bfs(g["sources"])
            outs.append(mesh.gs_diffuse(lv, float(g["t"]), 60)[0])
        o.set_threads(0)
    for u in outs:
        assert_same(u, g["u"])


TOL_CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "tol", "*.npz")))


@pytest.mark.parametrize("case", TOL_CASES)
def test_port_residual_tolerance_matches_reference(port_oracle, case):
    """DiffusionConfig::residual_tolerance early stop (diffusion.hpp:110-117)."""
    g = np.load(os.path.join(GOLDEN, "tol", case + ".npz"))
    mesh = port_oracle.build_mesh(g["positions"], g["faces"])
    lv = mesh.bfs(g["sources"])
    u, rep = mesh.gs_diffuse_tol(lv, float(g["t"]), int(g["sweeps"]), float(g["tolerance"]))
    assert rep.iterations == int(g["iterations"]) and rep.converged == bool(g["converged"])
    assert_same(u, g["u"], "u")
    assert_same(rep.primal_history, g["residual_history"], "E1 history")
