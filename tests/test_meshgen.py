"""Seeded mesh generators (CPU): identical to the reference generators where
they restate them, deterministic, and shaped as BASELINE.json describes."""
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1812_06060_b200 import meshgen


def test_mt19937_64_known_answer():
    # the C++ standard pins the 10000th output of default-seeded mt19937_64
    assert meshgen._load().gh_gen_mt64_first(5489) == 9981545732273789042


@pytest.mark.parametrize("case,gen", [("icosphere3", lambda: meshgen.icosphere(3)),
                                      ("icosphere5_config1", lambda: meshgen.icosphere(5)),
                                      ("torus60x30_three_sources", lambda: meshgen.torus(60, 30)[:2])])
def test_generators_match_reference_meshes(case, gen):
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    P, F = gen()
    assert np.array_equal(P.view(np.uint64), g["positions"].view(np.uint64))
    assert np.array_equal(F, g["faces"])


def test_config1_is_icosphere5():
    w = meshgen.config(1)
    g = np.load(os.path.join(GOLDEN, "icosphere5_config1.npz"))
    assert np.array_equal(w.positions, g["positions"]) and list(w.sources) == [0] and w.method == "face"


def test_config2_shape_and_determinism():
    a, b = meshgen.config(2, scale=32), meshgen.config(2, scale=32)
    n = 1024 // 32 + 1
    assert a.positions.shape == (n * n, 3) and a.faces.shape == (2 * (n - 1) ** 2, 3)
    assert np.array_equal(a.positions, b.positions)
    h = 1.0 / (n - 1)
    assert a.t == pytest.approx(h * h)
    # boundary vertices are not jittered; interior jitter is within +-0.2h
    P = a.positions.reshape(n, n, 3)
    ii, jj = np.meshgrid(np.arange(n), np.arange(n))
    assert np.array_equal(P[0, :, 1], np.zeros(n)) and np.allclose(P[:, 0, 0], 0)
    assert np.abs(P[..., 0] - ii * h).max() <= 0.2 * h + 1e-15
    assert np.abs(P[..., 2]).max() <= 0.08 + 1e-12
    # alternating diagonals: cell (0,0) splits along (0,0)-(1,1), cell (1,0) along (2,0)-(1,1)
    assert list(a.faces[0]) == [0, 1, n + 1] and list(a.faces[2]) == [1, 2, n + 1]


def test_config3_small_scale_torus():
    w = meshgen.config(3, scale=64)
    nu, nv = 4096 // 64, 2048 // 64
    assert w.positions.shape == (nu * nv, 3) and len(set(w.sources.tolist())) == 4
    # noise is along the tube normal, so |distance to tube circle - r| ~ N(0, (3e-4)^2)
    P = w.positions
    ring = np.hypot(P[:, 0], P[:, 1])
    dev = np.hypot(ring - 1.0, P[:, 2]) - 0.3
    assert 1e-4 < dev.std() < 6e-4 and np.abs(dev).max() < 3e-3


def test_config4_sh_displacement_bounds():
    w = meshgen.config(4, scale=256)  # icosphere level 3
    r = np.linalg.norm(w.positions, axis=1)
    assert r.min() >= 0.95 - 1e-12 and r.max() <= 1.05 + 1e-12
    assert max(abs(r.max() - 1.0), abs(r.min() - 1.0)) == pytest.approx(0.05, rel=1e-9)


def test_reference_arm_generator_build_matches():
    """bench.py --impl reference generates its workload with oracle/_ref's build
    of workloads/meshgen.c (so the reference process maps no product library):
    the arrays are bit-identical to the product build's, config by config."""
    import hashlib
    import subprocess
    import sys

    from conftest import ROOT
    from oracle import oracle as orc
    gen = os.path.join(orc.REF_DIR, "libgh_meshgen.so")
    if not os.path.exists(gen):
        orc.build()
    code = ("import sys, hashlib; sys.path.insert(0, %r)\n"
            "from paper_1812_06060_b200 import meshgen\n"
            "meshgen.use_library(%r)\n"
            "for k, s in ((1, 1), (2, 16), (3, 32), (4, 128), (5, 128)):\n"
            "    w = meshgen.config(k, scale=s)\n"
            "    print(hashlib.sha256(w.positions.tobytes() + w.faces.tobytes() + w.sources.tobytes()).hexdigest())\n"
            "print(meshgen._lib_path)\n") % (ROOT, gen)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, check=True).stdout.split()
    assert out[-1] == gen
    for (k, s), h in zip(((1, 1), (2, 16), (3, 32), (4, 128), (5, 128)), out):
        w = meshgen.config(k, scale=s)
        assert h == hashlib.sha256(w.positions.tobytes() + w.faces.tobytes() + w.sources.tobytes()).hexdigest(), k
