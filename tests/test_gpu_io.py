"""Mesh load -> device build on the GPU against the
reference loader and writers (mesh_io.hpp).

Every corpus file of tests/io_cases.py goes through gh_mesh_load_memory and
must end exactly where the reference ends (tests/golden/io_golden.json, made
from the reference): the same positions and faces on the device (sha256 of
their bytes), or the same exception text — parse errors, byte-offset
truncations, and build_mesh errors alike. Binary PLY records are decoded by
the device kernels; the report says so. Large meshes check the same
properties at scale: a binary PLY round trip is exact, and loading from a file
feeds the solver loop bit-identically to handing it the arrays.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import io_cases
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

IO_GOLDEN = json.load(open(os.path.join(GOLDEN, "io_golden.json")))
CASES = io_cases.all_cases()


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def _binary(fmt, data) -> bool:
    return fmt == io_cases.PLY and b"binary_little_endian" in data[:4096]


def _check(g, exp, load):
    if exp["ok"]:
        mesh, rep = load()
        P = mesh.download("positions").reshape(-1, 3)
        F = mesh.download("faces").reshape(-1, 3)
        assert (P.shape[0], F.shape[0]) == (exp["nv"], exp["nf"])
        assert sha(P) == exp["pos_sha"] and sha(F) == exp["faces_sha"]
        return rep
    with pytest.raises(g.MeshError) as ei:
        load()
    assert str(ei.value) == exp["error"]
    return None


@pytest.mark.parametrize("name,fmt,data", CASES, ids=[c[0] for c in CASES])
def test_load_memory_matches_reference(gpu, name, fmt, data):
    g = gpu.geoheat
    exp = IO_GOLDEN["cases"][name]
    rep = _check(g, exp, lambda: g.load_mesh(data, g.MeshFormat(fmt), with_report=True))
    if rep is not None:
        assert rep.bytes == len(data) and rep.binary == _binary(fmt, data)
        layout_fixed = not any(k in name for k in ("vertex_list", "two_face_lists", "third_face"))
        if rep.binary and exp["nv"] and layout_fixed:
            assert rep.device_decoded and rep.kernel_launches > 0


def test_load_from_path(gpu, tmp_path):
    g = gpu.geoheat
    for name in ("obj_square_crlf_tabs_comments", "ply_ascii_grid10x7", "ply_bin_grid16x11", "ply_bin_mixed_types",
                 "ply_bin_truncated_mid_face", "obj_face_index_out_of_range"):
        fmt, data = next((f, d) for n, f, d in CASES if n == name)
        p = tmp_path / (name + (".obj" if fmt == io_cases.OBJ else ".PLY"))
        p.write_bytes(data)
        _check(g, IO_GOLDEN["cases"][name], lambda: g.load_mesh(str(p), with_report=True))
    with pytest.raises(g.MeshError, match="cannot open mesh file '.*missing.obj'"):
        g.load_mesh(str(tmp_path / "missing.obj"))
    with pytest.raises(g.MeshError, match="cannot infer mesh format from path"):
        g.load_mesh(str(tmp_path / "mesh.stl"))


@pytest.mark.parametrize("name", sorted(IO_GOLDEN["writers"]))
def test_writers_match_reference(gpu, name, tmp_path):
    g = gpu.geoheat
    w = IO_GOLDEN["writers"][name]
    P, F = io_cases.grid(w["nx"], w["ny"], jitter=w["jitter"], seed=w["seed"])
    mesh = g.build_mesh(P, F)
    q = np.sqrt(np.arange(P.shape[0], dtype=np.float64)) * 0.7
    h = lambda b: hashlib.sha256(b).hexdigest()[:32]  # noqa: E731
    assert h(g.serialize_mesh(mesh, g.MeshFormat.OBJ)) == w["obj_sha"]
    assert h(g.serialize_mesh(mesh, g.MeshFormat.PLY)) == w["ply_sha"]
    assert h(g.serialize_mesh(mesh, g.MeshFormat.PLY, q)) == w["ply_quality_sha"]
    g.save_mesh(str(tmp_path / "m.ply"), mesh, q)
    assert h((tmp_path / "m.ply").read_bytes()) == w["ply_quality_sha"]
    g.save_mesh(str(tmp_path / "m.obj"), mesh)
    back = g.load_mesh(str(tmp_path / "m.obj"))  # %.17g round-trips (test_io.cpp OBJ round trip)
    assert np.array_equal(back.download("positions").reshape(-1, 3), P)
    with pytest.raises(ValueError):
        g.save_mesh(str(tmp_path / "q.obj"), mesh, q)
    with pytest.raises(g.MeshError, match="cannot infer mesh format"):
        g.save_mesh(str(tmp_path / "m.stl"), mesh)


def _binary_ply(P, F) -> bytes:
    vt = np.dtype([("x", "<f8"), ("y", "<f8"), ("z", "<f8")])
    ft = np.dtype([("n", "u1"), ("i", "<i4", (3,))])
    V = np.empty(P.shape[0], vt)
    V["x"], V["y"], V["z"] = P[:, 0], P[:, 1], P[:, 2]
    Fr = np.empty(F.shape[0], ft)
    Fr["n"] = 3
    Fr["i"] = F
    head = ("ply\nformat binary_little_endian 1.0\nelement vertex %d\nproperty double x\nproperty double y\n"
            "property double z\nelement face %d\nproperty list uchar int vertex_indices\nend_header\n"
            % (P.shape[0], F.shape[0])).encode()
    return head + V.tobytes() + Fr.tobytes()


def test_large_binary_ply_round_trip_and_solve(gpu, tmp_path):
    """1.05M vertices: file -> device decode -> build is exact, the solver loop
    from the loaded mesh equals the one from the arrays, and save_ply writes
    the same bytes the numpy packer produced."""
    g = gpu.geoheat
    from paper_1812_06060_b200 import meshgen
    w = meshgen.config(2, scale=1)
    data = _binary_ply(w.positions, w.faces)
    p = tmp_path / "c2.ply"
    p.write_bytes(data)
    mesh, rep = g.load_mesh(str(p), with_report=True)
    assert rep.device_decoded and rep.binary
    assert np.array_equal(mesh.download("positions").reshape(-1, 3), w.positions)
    assert np.array_equal(mesh.download("faces").reshape(-1, 3), w.faces)
    assert g.serialize_mesh(mesh, g.MeshFormat.PLY) == data
    levels = g.bfs_levels(mesh, w.sources)
    d_file, _ = g.distance(levels, method=w.method, sweeps=50, t=w.t)
    d_arr, _ = g.distance_host(w.positions, w.faces, w.sources, method=w.method, sweeps=50, t=w.t)
    assert np.array_equal(d_file, d_arr)
    # truncating the body anywhere in the faces reports the reference's offset
    head = data.index(b"end_header\n") + 11
    cut = head + 24 * w.positions.shape[0] + 13 * 777_777 + 5
    with pytest.raises(g.MeshError, match="byte offset %d: unexpected end of data" % (cut - head)):
        g.load_mesh(data[:cut], g.MeshFormat.PLY)
    # a bad record deep in the body is found by the decoder and worded exactly
    bad = bytearray(data)
    bad[head + 24 * w.positions.shape[0] + 13 * 1_500_000] = 4
    with pytest.raises(g.MeshError, match="PLY: non-triangle face with 4 vertices"):
        g.load_mesh(bytes(bad), g.MeshFormat.PLY)


def test_large_text_formats(gpu):
    g = gpu.geoheat
    P, F = io_cases.grid(400, 300, jitter=0.1, seed=4)
    for fmt, data in ((g.MeshFormat.OBJ, io_cases.obj_text(P, F)), (g.MeshFormat.PLY, io_cases.ply_ascii(P, F))):
        mesh, rep = g.load_mesh(data, fmt, with_report=True)
        assert not rep.device_decoded and rep.host_threads >= 1
        assert np.array_equal(mesh.download("positions").reshape(-1, 3), P)
        assert np.array_equal(mesh.download("faces").reshape(-1, 3), F)
