"""Mesh I/O host logic (CPU): the text tokenisers (OBJ, ASCII PLY) and the
writers against the reference loader / writers (mesh_io.hpp).

Golden outcomes (tests/golden/io_golden.json, made by make_io_golden.py from
the reference itself) pin every corpus file of tests/io_cases.py: the exact
positions/faces or the exact exception text. A reference failure that comes
from build_mesh (not the parser) must leave our tokeniser's output such that
build_mesh (the port oracle's restatement) raises that same text. When the
compiled reference is present, a second seeded fuzz corpus is checked live.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import io_cases
from conftest import GOLDEN
from paper_1812_06060_b200 import geoheat as g

IO_GOLDEN = json.load(open(os.path.join(GOLDEN, "io_golden.json")))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def _is_text(fmt, data) -> bool:
    if fmt == io_cases.OBJ:
        return True
    head = data[:4096]
    return b"binary_little_endian" not in head


def _parse(fmt, data, threads=0):
    try:
        P, F = g.parse_mesh_text(data, g.MeshFormat(fmt), threads)
        return True, (P, F)
    except g.MeshError as e:
        return False, str(e)
    except ValueError as e:  # binary PLY handed to the text tokeniser
        return None, str(e)


def _check_against(expected, fmt, data, port_oracle, threads=0):
    ok, res = _parse(fmt, data, threads)
    if ok is None:
        pytest.fail(f"binary body reached the text tokeniser: {res}")
    if expected["ok"]:
        assert ok, f"reference loads, ours raised: {res}"
        P, F = res
        assert (P.shape[0], F.shape[0]) == (expected["nv"], expected["nf"])
        assert sha(P) == expected["pos_sha"] and sha(F.astype(np.int32)) == expected["faces_sha"]
        return
    if not ok:
        assert res == expected["error"]
        return
    # the reference failed in build_mesh: our tokens must fail there identically
    P, F = res
    from oracle.oracle import OracleMeshError
    with pytest.raises(OracleMeshError) as ei:
        port_oracle.build_mesh(P, F)
    assert str(ei.value) == expected["error"]


TEXT_CASES = [(n, f, d) for n, f, d in io_cases.all_cases() if _is_text(f, d)]


def test_corpus_matches_golden_inputs():
    cases = io_cases.all_cases()
    assert len(cases) == len(IO_GOLDEN["cases"])
    for name, fmt, data in cases:
        rec = IO_GOLDEN["cases"][name]
        assert rec["format"] == fmt and rec["data_sha"] == hashlib.sha256(data).hexdigest()[:32], name


@pytest.mark.parametrize("name,fmt,data", TEXT_CASES, ids=[c[0] for c in TEXT_CASES])
def test_text_parse_matches_reference(name, fmt, data, port_oracle):
    _check_against(IO_GOLDEN["cases"][name], fmt, data, port_oracle)


@pytest.mark.parametrize("threads", [1, 2, 3, 7])
def test_thread_count_does_not_change_result(threads, port_oracle):
    # line-aligned chunks: first-error-wins and relative indices across chunk cuts
    for name, fmt, data in TEXT_CASES:
        if len(data) > 300 or name.startswith("fuzz"):
            _check_against(IO_GOLDEN["cases"][name], fmt, data, port_oracle, threads)


def test_large_obj_many_threads_matches_single():
    P, F = io_cases.grid(120, 90, jitter=0.2, seed=9)
    data = io_cases.obj_text(P, F)
    a = g.parse_mesh_text(data, g.MeshFormat.OBJ, 1)
    b = g.parse_mesh_text(data, g.MeshFormat.OBJ, 16)
    assert np.array_equal(a[0], P) and np.array_equal(a[1], F)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # an error deep in the file is reported at its line whatever the split
    lines = data.split(b"\n")
    bad_line = len(P) + 1000
    lines[bad_line - 1] = b"f 1 2 %d" % (len(P) + 5)
    bad = b"\n".join(lines)
    for t in (1, 5, 16):
        with pytest.raises(g.MeshError, match=f"at line {bad_line}: face index out of range"):
            g.parse_mesh_text(bad, g.MeshFormat.OBJ, t)


def test_binary_ply_is_not_tokenised_on_host():
    with pytest.raises(ValueError, match="decoded on the device"):
        g.parse_mesh_text(io_cases.square_binary(), g.MeshFormat.PLY)


def test_format_from_path():
    # test_io.cpp "format inference"
    assert g.format_from_path("a/b/mesh.obj") == g.MeshFormat.OBJ
    assert g.format_from_path("MESH.PLY") == g.MeshFormat.PLY
    with pytest.raises(g.MeshError, match="cannot infer mesh format from path 'mesh.stl'"):
        g.format_from_path("mesh.stl")


@pytest.mark.parametrize("name", sorted(IO_GOLDEN["distances"]))
@pytest.mark.parametrize("csv", [False, True])
def test_distance_writers_match_reference(name, csv):
    rec = IO_GOLDEN["distances"][name]
    vec = np.array([float(v) for v in rec["values"]])
    assert g.format_distances(vec, csv=csv).decode() == rec["csv" if csv else "txt"]


def test_distance_writers_large_parallel(tmp_path):
    rng = np.random.RandomState(3)
    d = rng.standard_normal(300_000) * 10.0 ** rng.randint(-30, 30, 300_000)
    txt = g.format_distances(d)
    parsed = np.array([float(x) for x in txt.decode().split()])
    assert np.array_equal(parsed, d)  # %.17g round-trips (test_io.cpp "distance writers")
    p = tmp_path / "d.csv"
    g.write_distances(str(p), d[:1000], csv=True)
    assert p.read_bytes() == g.format_distances(d[:1000], csv=True)


def _ref_oracle():
    from oracle.oracle import Oracle, available
    if not available("reference"):
        pytest.skip("compiled reference (oracle/_ref/libgeoheat_ref.so) not present")
    return Oracle("reference")


def test_live_fuzz_against_reference(port_oracle):
    o = _ref_oracle()
    from oracle.oracle import OracleMeshError
    cases = io_cases.fuzz_cases(seed=20260601, n_text=600, n_bin=0)
    for name, fmt, data in cases:
        if not _is_text(fmt, data):
            continue
        try:
            m = o.load_mesh(data, fmt)
            P = m.array("positions").reshape(-1, 3)
            F = m.array("faces").reshape(-1, 3)
            exp = {"ok": True, "nv": P.shape[0], "nf": F.shape[0], "pos_sha": sha(P), "faces_sha": sha(F)}
        except OracleMeshError as e:
            exp = {"ok": False, "error": str(e)}
        _check_against(exp, fmt, data, port_oracle, threads=1 + len(data) % 4)


def test_number_grammar_against_reference(port_oracle):
    """std::istream >> double corner cases, one vertex coordinate at a time."""
    o = _ref_oracle()
    from oracle.oracle import OracleMeshError
    rng = np.random.RandomState(7)
    pieces = ["0", "1", "9", ".", "e", "E", "+", "-", "00", "5", "x", "p", "inf", "nan", "1e308", "9e-324", "7"]
    for _ in range(1500):
        tok = "".join(pieces[rng.randint(len(pieces))] for _ in range(1 + rng.randint(5)))
        data = ("v %s 0 0\nv 1 0 0 \nv 0 1 0\nf 1 2 3\n" % tok).encode()
        try:
            m = o.load_mesh(data, 0)
            P = m.array("positions").reshape(-1, 3)
            F = m.array("faces").reshape(-1, 3)
            exp = {"ok": True, "nv": P.shape[0], "nf": F.shape[0], "pos_sha": sha(P), "faces_sha": sha(F)}
        except OracleMeshError as e:
            exp = {"ok": False, "error": str(e)}
        _check_against(exp, 0, data, port_oracle)
