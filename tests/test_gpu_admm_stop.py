"""The ADMM stop rule (grad_face.hpp:175-177, grad_edge.hpp:168-170) decided on
the device: iteration counts, converged flags, histories and outputs equal the
C oracle's when the rule fires early, never fires, fires at the first
iteration, and when a threshold sits exactly on a residual norm (inside the
guard band, where the device halts and the host decides from the exact
left-to-right sums)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torus(gpu, port_oracle):
    from paper_1812_06060_b200 import meshgen
    w = meshgen.config(3, scale=16)  # closed 256 x 128 torus: every edge interior
    om = port_oracle.build_mesh(w.positions, w.faces)
    lv = om.bfs(w.sources)
    t = om.diffusion_time(1.0)
    u, _ = om.gs_diffuse(lv, t, 300)
    H, _ = om.normalized_target_gradients(u)
    mesh = gpu.build_mesh(w.positions, w.faces)
    P, F = w.positions, w.faces
    area = 0.5 * np.linalg.norm(np.cross(P[F[:, 1]] - P[F[:, 0]], P[F[:, 2]] - P[F[:, 0]]), axis=1)
    return dict(om=om, mesh=mesh, H=H, face_scale=np.sqrt(3.0 * area.sum()), edge_scale=np.sqrt(3.0 * len(F)))


def _run(gpu, torus, method, iters, eps1, eps2):
    cfg = gpu.AdmmConfig(max_iterations=iters, eps1=eps1, eps2=eps2)
    if method == "face":
        r = gpu.admm_face_optimize(torus["mesh"], torus["H"], cfg)
        out, rep = r.gradients, r.report
        ref, rrep = torus["om"].admm_face(torus["H"], iters, eps1, eps2)
    else:
        r = gpu.admm_edge_optimize(torus["mesh"], torus["H"], cfg)
        out, rep = r.differences, r.report
        ref, rrep = torus["om"].admm_edge(torus["H"], iters, eps1, eps2)
    assert rep.iterations == rrep.iterations and rep.converged == rrep.converged, (method, eps1, eps2)
    assert np.array_equal(np.asarray(out).view(np.uint64), np.asarray(ref).view(np.uint64))
    np.testing.assert_allclose(rep.primal_history, rrep.primal_history, rtol=1e-12)
    np.testing.assert_allclose(rep.dual_history, rrep.dual_history, rtol=1e-12)
    return rep


@pytest.mark.parametrize("method", ["face", "edge"])
def test_stop_rule_cases(gpu, torus, method):
    # never / at the first iteration
    rep = _run(gpu, torus, method, 12, 1e-30, 1e-30)
    assert rep.iterations == 12 and not rep.converged
    rep = _run(gpu, torus, method, 12, 1e30, 1e30)
    assert rep.iterations == 1 and rep.converged
    # thresholds between two iterations' residuals: stops in the middle, in
    # the first batch of enqueued iterations or a later one (16 per batch)
    full = _run(gpu, torus, method, 60, 1e-30, 1e-30)
    scale = torus["face_scale" if method == "face" else "edge_scale"]
    for k in (6, 20, 40):
        eps1 = full.primal_history[k] / scale * (1 + 1e-6)  # iteration k meets both
        eps2 = full.dual_history[k] / scale * (1 + 1e-6)
        rep = _run(gpu, torus, method, 60, eps1, eps2)
        assert rep.converged and rep.iterations <= k + 1


@pytest.mark.parametrize("method", ["face", "edge"])
@pytest.mark.parametrize("k", [0, 3, 7])
def test_threshold_on_a_residual(gpu, torus, method, k):
    """eps chosen so scale * eps equals iteration k's residual to a few ulps:
    the device halts in the guard band, the exact sums decide, and whatever
    they decide (stop or continue) matches the reference."""
    full = _run(gpu, torus, method, 12, 1e-30, 1e-30)
    scale = torus["face_scale" if method == "face" else "edge_scale"]
    for j, (p, d) in enumerate(zip(full.primal_history, full.dual_history)):
        if j != k:
            continue
        _run(gpu, torus, method, 12, p / scale, 1e30)   # primal on its threshold
        _run(gpu, torus, method, 12, 1e30, d / scale)   # dual on its threshold
        _run(gpu, torus, method, 12, p / scale, d / scale)
