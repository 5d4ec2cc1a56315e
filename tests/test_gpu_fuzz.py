"""Seeded random meshes through the whole chain, GPU vs the compiled reference
(oracle/_ref): ragged grids with holes and isolated vertices (unreachable
vertices, several components), duplicate sources, zero sweeps / iterations,
both optimisers — every stage bit-identical — and corrupted meshes (flipped
winding, duplicated face, out-of-range index, repeated vertex, collinear
face) rejected with the reference's exact message.
"""
import numpy as np
import pytest

import io_cases

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref():
    from oracle.oracle import Oracle, available
    assert available("reference"), "oracle/_ref/libgeoheat_ref.so missing"
    return Oracle("reference")


def _random_mesh(rng):
    nx, ny = rng.randint(2, 40), rng.randint(2, 30)
    P, F = io_cases.grid(nx, ny, jitter=rng.uniform(0, 0.3), seed=int(rng.randint(1 << 30)))
    P[:, :2] += rng.uniform(-0.2, 0.2, (P.shape[0], 2)) / max(nx, ny)
    keep = rng.uniform(size=F.shape[0]) >= rng.uniform(0.0, 0.25)
    keep[0] = True
    return P, F[keep]


def _corrupt(rng, P, F):
    F = F.copy()
    kind = rng.randint(5)
    f = rng.randint(F.shape[0])
    if kind == 0:
        F[f] = F[f][::-1]                       # flipped winding
    elif kind == 1:
        F = np.vstack([F, F[f:f + 1]])           # duplicated face: non-manifold edges
    elif kind == 2:
        F[f, rng.randint(3)] = P.shape[0] + rng.randint(5)  # index out of range
    elif kind == 3:
        F[f, 1] = F[f, 0]                        # repeated vertex
    else:
        a, b = F[f, 0], F[f, 1]                  # collinear: third corner on the line a-b
        P = P.copy()
        P[F[f, 2]] = 0.5 * (P[a] + P[b])
    return P, F


@pytest.mark.parametrize("seed", range(24))
def test_random_chain_bitwise(gpu, ref, seed):
    g = gpu.geoheat
    from oracle.oracle import OracleMeshError
    rng = np.random.RandomState(1812060600 + 97 * seed)
    P, F = _random_mesh(rng)
    try:
        om = ref.build_mesh(P, F)
    except OracleMeshError as e:
        with pytest.raises(g.MeshError) as ei:
            g.build_mesh(P, F)
        assert str(ei.value) == str(e)
        return
    mesh = g.build_mesh(P, F)
    for name in ("faces", "edge_vertices", "halfedge_twin", "interior_edges", "vertex_area", "halfedge_cot",
                 "edge_weight", "vv_offset", "vv_index", "vv_weight"):
        assert np.array_equal(mesh.download(name).ravel(), om.array(name).ravel()), name
    used = np.unique(F)
    sources = list(rng.choice(used, size=rng.randint(1, 5)))  # duplicates allowed
    sweeps = int(rng.choice([0, 1, 7, 60, 200]))
    iters = int(rng.choice([0, 1, 5, 20]))
    t = om.diffusion_time(float(rng.choice([0.5, 1.0, 4.0])))
    olv = om.bfs(sources)
    lv = g.bfs_levels(mesh, sources)
    assert np.array_equal(lv.level_of_vertex, olv.level_of_vertex)
    assert np.array_equal(lv.parent_of_vertex, olv.parent_of_vertex)
    assert lv.unreachable_count == int((olv.level_of_vertex < 0).sum())
    u_ref, _ = om.gs_diffuse(olv, t, sweeps)
    u = g.gs_diffuse(mesh, lv, t, g.DiffusionConfig(sweeps=sweeps))
    assert np.array_equal(u, u_ref)
    H_ref, zc_ref = om.normalized_target_gradients(u_ref)
    nt = g.normalized_target_gradients(mesh, u)
    assert np.array_equal(nt.field, H_ref) and nt.zero_count == zc_ref
    G_ref, fr = om.admm_face(H_ref, iters)
    fres = g.admm_face_optimize(mesh, nt.field, g.AdmmConfig(max_iterations=iters))
    assert fres.report.iterations == fr.iterations and fres.report.converged == fr.converged
    assert np.array_equal(fres.gradients, G_ref)
    X_ref, er = om.admm_edge(H_ref, iters)
    eres = g.admm_edge_optimize(mesh, nt.field, g.AdmmConfig(max_iterations=iters))
    assert eres.report.iterations == er.iterations and eres.report.converged == er.converged
    assert np.array_equal(eres.differences, X_ref)
    assert np.array_equal(g.integrate_face_gradients(mesh, lv, fres.gradients), om.integrate_face(olv, G_ref))
    assert np.array_equal(g.integrate_edge_differences(mesh, lv, eres.differences), om.integrate_edge(olv, X_ref))


@pytest.mark.parametrize("seed", range(30))
def test_corrupted_mesh_messages(gpu, ref, seed):
    g = gpu.geoheat
    from oracle.oracle import OracleMeshError
    rng = np.random.RandomState(20261020 + seed)
    P, F = _random_mesh(rng)
    P, F = _corrupt(rng, P, F)
    try:
        ref.build_mesh(P, F)
    except OracleMeshError as e:
        with pytest.raises(g.MeshError) as ei:
            g.build_mesh(P, F)
        assert str(ei.value) == str(e)
        return
    g.build_mesh(P, F)  # the corruption happened to be harmless for the reference too
