"""The CG heat method and the evaluation layer on the device (SURVEY §8(f)
rows 3-4) against the compiled reference (oracle/_ref, built from
/root/reference; it ships with the repo snapshot).

  poisson_heat_method   reference.hpp:175-216 — distances to 1e-9 relative,
                        same CG iteration counts (dot products are tree sums
                        here, left-to-right there)
  dijkstra_edge_distance reference.hpp:220-245 — bit-identical
  midpoint_subdivide    subdivide.hpp:14-44 — bit-identical meshes
  analytic_oracle       reference.hpp:283-321 — plane bit-identical, sphere
                        to 1e-12 (centre/radius are tree sums, acos differs)
  triangulation_quality, mean_relative_error, recovery_error — bit-identical
                        (left-to-right sums reproduced exactly, gh_seqsum.cu)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

MESHES = [
    ("hex_disk", (12,), [0, 7]),
    ("icosphere", (3,), [0]),
    ("torus", (24, 12), [5, 100]),
    ("grid", (16, 11), [0]),
    ("uv_sphere", (8, 16), [3]),
    ("two_disjoint_triangles", (), [0]),
    ("strip", (40,), [0, 41]),
]


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    assert available("reference"), "oracle/_ref/libgeoheat_ref.so missing (built by __graft_entry__.build())"
    return Oracle("reference")


def _meshes(gpu, ref, name, params):
    P, F = ref.test_mesh(name, *params)
    return P, F, gpu.geoheat.build_mesh(P, F), ref.build_mesh(P, F)


@pytest.mark.parametrize("name,params,sources", MESHES, ids=[m[0] for m in MESHES])
def test_poisson_heat_method_matches_reference(gpu, ref, name, params, sources):
    g = gpu.geoheat
    P, F, mesh, om = _meshes(gpu, ref, name, params)
    t = om.diffusion_time(1.0)
    d_ref, it_ref, res_ref = ref.poisson(om, sources, t, 1e-5)
    d, rep = g.poisson_heat_method(mesh, sources, t, 1e-5)
    assert (rep.heat_iterations, rep.poisson_iterations) == it_ref
    fin = np.isfinite(d_ref)
    assert np.array_equal(fin, np.isfinite(d)) and np.array_equal(d[~fin], d_ref[~fin])
    scale = max(1.0, np.abs(d_ref[fin]).max())
    assert np.max(np.abs(d[fin] - d_ref[fin])) <= 1e-9 * scale
    assert rep.poisson_residual == pytest.approx(res_ref[1], rel=1e-6, abs=1e-15)
    # the same solve through the fused pipeline entry point (method "poisson")
    levels = g.bfs_levels(mesh, sources)
    d2, r2 = g.distance(levels, method="poisson", t=t, cg_tol=1e-5)
    assert np.array_equal(d, d2) and r2.cg_iterations == sum(it_ref)


def test_poisson_tight_tolerance_and_breakdown_free(gpu, ref):
    g = gpu.geoheat
    P, F, mesh, om = _meshes(gpu, ref, "hex_disk", (20,))
    t = om.diffusion_time(1.0)
    d_ref, it_ref, _ = ref.poisson(om, [0], t, 1e-10)
    d, rep = g.poisson_heat_method(mesh, [0], t, 1e-10)
    assert abs(rep.heat_iterations - it_ref[0]) <= 1 and abs(rep.poisson_iterations - it_ref[1]) <= 1
    assert np.max(np.abs(d - d_ref)) <= 1e-10 * np.abs(d_ref).max()


@pytest.mark.parametrize("name,params,sources", MESHES, ids=[m[0] for m in MESHES])
def test_dijkstra_bitwise(gpu, ref, name, params, sources):
    P, F, mesh, om = _meshes(gpu, ref, name, params)
    assert np.array_equal(gpu.geoheat.dijkstra_edge_distance(mesh, sources), ref.dijkstra(om, sources))


@pytest.mark.parametrize("levels", [0, 1, 2])
@pytest.mark.parametrize("name,params", [("unit_square", ()), ("hex_disk", (5,)), ("icosphere", (1,)),
                                         ("torus", (12, 6))])
def test_subdivide_bitwise(gpu, ref, name, params, levels):
    P, F, mesh, om = _meshes(gpu, ref, name, params)
    fine = gpu.geoheat.midpoint_subdivide(mesh, levels)
    ofine = ref.subdivide(om, levels)
    for arr in ("positions", "faces", "edge_vertices", "vertex_area", "halfedge_cot"):
        assert np.array_equal(fine.download(arr).ravel(), ofine.array(arr).ravel()), arr


def test_quality_analytic_and_error_metrics(gpu, ref):
    g = gpu.geoheat
    for name, params in (("hex_disk", (15,)), ("icosphere", (4,)), ("torus", (30, 14)), ("grid", (20, 9))):
        P, F, mesh, om = _meshes(gpu, ref, name, params)
        assert g.triangulation_quality(mesh) == om.triangulation_quality()  # left-to-right sum, bit for bit
    # plane: bit-identical; multi-source pointwise minimum
    P, F, mesh, om = _meshes(gpu, ref, "hex_disk", (15,))
    dp = g.analytic_oracle(g.AnalyticSurface.PlaneEuclidean, mesh, [0, 40])
    assert np.array_equal(dp, om.analytic(0, [0, 40]))
    with pytest.raises(ValueError, match="not on a common sphere"):
        g.analytic_oracle(g.AnalyticSurface.SphereGreatCircle, mesh, [0])
    # sphere
    P, F, mesh, om = _meshes(gpu, ref, "icosphere", (4,))
    ds = g.analytic_oracle(g.AnalyticSurface.SphereGreatCircle, mesh, [0, 17])
    np.testing.assert_allclose(ds, om.analytic(1, [0, 17]), rtol=1e-12, atol=1e-15)
    with pytest.raises(ValueError, match="not planar"):
        g.analytic_oracle(g.AnalyticSurface.PlaneEuclidean, mesh, [0])
    # error metrics on a solved field, with excluded vertices (zero / inf refs)
    d, _ = g.distance(g.bfs_levels(mesh, [0]), method="edge", sweeps=200, m=1.0)
    r = ds.copy()
    r[5] = 0.0
    r[9] = np.inf
    mre, exc, e2 = g.error_metrics(d, r, [0, 17])
    assert mre == om.mean_relative_error(d, r, [0, 17])
    assert exc == ref.mre_excluded(d, r, [0, 17])
    rfin = ds
    _, _, e2 = g.error_metrics(d, rfin, [0])
    assert e2 == ref.recovery_error(d, rfin)


def test_pipeline_diffusion_e1(gpu, ref):
    g = gpu.geoheat
    P, F, mesh, om = _meshes(gpu, ref, "torus", (24, 12))
    levels = g.bfs_levels(mesh, [5])
    t = om.diffusion_time(1.0)
    d, rep = g.distance(levels, method="face", sweeps=40, t=t, diffusion_e1=True)
    u = g.gs_diffuse(mesh, levels, t, g.DiffusionConfig(sweeps=40))
    assert rep.diffusion_e1 == g.diffusion_residual(mesh, u, t, [5], levels)
    assert rep.diffusion_e1 == pytest.approx(om.diffusion_residual(u, t, [5]), rel=1e-12)
    _, rep0 = g.distance(levels, method="face", sweeps=40, t=t)
    assert rep0.diffusion_e1 == -1.0
