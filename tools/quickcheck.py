"""Developer quick check: GPU path vs the C oracle on a few small meshes (bitwise)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1812_06060_b200 as gh
from paper_1812_06060_b200 import meshgen
from oracle.oracle import Oracle

o = Oracle("port")
fails = 0
def same(a, b):
    a = np.asarray(a); b = np.asarray(b)
    if a.dtype == np.float64:
        return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))
    return a.shape == b.shape and np.array_equal(a, b)

cases = []
P, F = meshgen.icosphere(3); cases.append(("ico3", P, F, [0], 50))
P, F, S = meshgen.torus(64, 32, 1.0, 0.3, 1e-3 * 0.3, 7, 4); cases.append(("torus64", P, F, S, 100))
P, F = meshgen.grid(33, 0.2, 0.02, 3); cases.append(("grid33", P, F, [16 * 33 + 16], 200))
P, F = meshgen.icosphere(5); cases.append(("ico5", P, F, [0], 1000))
for name, P, F, S, sweeps in cases:
    om = o.build_mesh(P, F)
    t0 = time.time()
    m = gh.build_mesh(P, F)
    tb = time.time() - t0
    bad = [a for a, *_ in gh.geoheat.MESH_ARRAYS if not same(m.download(a).ravel(), om.array(a).ravel())]
    ol = om.bfs(S)
    lv = gh.bfs_levels(m, S)
    bfs_ok = same(lv.level_of_vertex, ol.level_of_vertex) and same(lv.parent_of_vertex, ol.parent_of_vertex) and same(lv.order, ol.order) and same(lv.offsets, ol.offsets)
    t = om.diffusion_time(1.0)
    tg = gh.diffusion_time(m, 1.0)
    uo, _ = om.gs_diffuse(ol, t, sweeps)
    rep = gh.SolverReport()
    u = gh.gs_diffuse(m, lv, t, gh.DiffusionConfig(sweeps=sweeps), rep)
    Ho, zo = om.normalized_target_gradients(uo)
    nh = gh.normalized_target_gradients(m, uo)
    Go, ro = om.admm_face(Ho)
    fr = gh.admm_face_optimize(m, Ho)
    Xo, reo = om.admm_edge(Ho)
    er = gh.admm_edge_optimize(m, Ho)
    do = om.integrate_face(ol, Go); d = gh.integrate_face_gradients(m, lv, Go)
    deo = om.integrate_edge(ol, Xo); de = gh.integrate_edge_differences(m, lv, Xo)
    dd, rr = gh.distance(lv, "face", sweeps, t)
    res = dict(mesh=not bad, bfs=bfs_ok, t_rel=abs(tg - t) / t, u=same(u, uo), H=same(nh.field, Ho), zc=(nh.zero_count, zo),
               G=same(fr.gradients, Go), it=(fr.report.iterations, ro.iterations),
               primal=max(abs(a - b) / b for a, b in zip(fr.report.primal_history, ro.primal_history)),
               X=same(er.differences, Xo), de=same(de, deo), d=same(d, do), fused=same(dd, do))
    ok = all(v for k, v in res.items() if isinstance(v, bool))
    fails += not ok
    print(name, "OK" if ok else "FAIL", res, "bad arrays:", bad, "diff_ms=%.3f build_s=%.3f" % (rep.device_ms, tb))
print("done", flush=True)
pass
print("freed", flush=True)
sys.exit(1 if fails else 0)
