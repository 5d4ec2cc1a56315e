"""Reference outcomes for the mesh I/O corpus (tests/io_cases.py).

Runs the UNMODIFIED reference loader and writers (mesh_io.hpp via
oracle/_ref/libgeoheat_ref.so, built from /root/reference by
oracle/build_ref.sh) on every corpus file and records what it returns: the
positions/faces it hands out (sha256 of their bytes) or the exact exception
text. Writers: the bytes of save_obj / save_ply (with and without quality)
and write_distances_txt / _csv. Needs /root/reference, so it runs in the
build container only; io_golden.json is committed and travels.

    python tests/golden/make_io_golden.py
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle.oracle import Oracle, OracleMeshError  # noqa: E402
import io_cases  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:32]


def outcome(o: Oracle, fmt: int, data: bytes) -> dict:
    try:
        m = o.load_mesh(data, fmt)
    except OracleMeshError as e:
        return {"ok": False, "error": str(e)}
    P = m.array("positions").reshape(-1, 3)
    F = m.array("faces").reshape(-1, 3)
    return {"ok": True, "nv": int(P.shape[0]), "nf": int(F.shape[0]), "pos_sha": sha(P), "faces_sha": sha(F)}


WRITER_MESHES = [("grid9x5", 9, 5, 0.3, 21), ("grid1x1", 1, 1, 0.0, 0)]
DISTANCE_VECTORS = {
    "test_io": [0.0, 1.0 / 3.0, 2.0 ** 0.5, float("inf")],
    "mixed": [-0.0, 1e-300, 5e-324, 1.7976931348623157e308, 123456789.125, -2.5, float("nan"), 0.1],
}


def main() -> None:
    o = Oracle("reference")
    cases = {}
    for name, fmt, data in io_cases.all_cases():
        assert name not in cases, name
        rec = {"format": fmt, "data_sha": hashlib.sha256(data).hexdigest()[:32], "bytes": len(data)}
        rec.update(outcome(o, fmt, data))
        cases[name] = rec
    writers = {}
    for name, nx, ny, jit, seed in WRITER_MESHES:
        P, F = io_cases.grid(nx, ny, jitter=jit, seed=seed)
        m = o.build_mesh(P, F)
        q = np.sqrt(np.arange(P.shape[0], dtype=np.float64)) * 0.7
        writers[name] = {
            "nx": nx, "ny": ny, "jitter": jit, "seed": seed,
            "obj_sha": hashlib.sha256(o.save_mesh(m, 0)).hexdigest()[:32],
            "ply_sha": hashlib.sha256(o.save_mesh(m, 1)).hexdigest()[:32],
            "ply_quality_sha": hashlib.sha256(o.save_mesh(m, 1, q)).hexdigest()[:32],
        }
    dist = {}
    for name, vec in DISTANCE_VECTORS.items():
        dist[name] = {"values": [repr(v) for v in vec],
                      "txt": o.write_distances(np.asarray(vec), False).decode(),
                      "csv": o.write_distances(np.asarray(vec), True).decode()}
    out = {"generator": "tests/golden/make_io_golden.py", "cases": cases, "writers": writers, "distances": dist}
    with open(os.path.join(HERE, "io_golden.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    n_ok = sum(1 for c in cases.values() if c["ok"])
    print(f"{len(cases)} cases ({n_ok} load, {len(cases) - n_ok} raise); {len(writers)} writer meshes")


if __name__ == "__main__":
    main()
