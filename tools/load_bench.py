"""Mesh load -> device build timing.

Writes the BASELINE config meshes as binary PLY and OBJ (with this repo's
own writers), then times gh_mesh_load(path) -> device TriMesh ready for BFS:
file mapping, host->device staging, record decode / tokenising, build_mesh.
Files sit in the page cache (just written), so this is the warm-cache load.
The reference loader (load_mesh + build_mesh, mesh_io.hpp via the compiled
reference in oracle/_ref) is timed beside it on the config-2 mesh.

    python tools/load_bench.py [--configs 2,3] [--out gpurun_out/load.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1812_06060_b200 import geoheat as g  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402


def time_load(path: str, reps: int = 3):
    best = None
    for _ in range(reps):
        t0 = time.perf_counter()
        mesh, rep = g.load_mesh(path, with_report=True)
        wall = (time.perf_counter() - t0) * 1e3
        if best is None or wall < best[0]:
            best = (wall, rep, mesh.vertex_count(), mesh.face_count())
        del mesh
    wall, rep, nv, nf = best
    return {"wall_ms": wall, "read_ms": rep.read_ms, "parse_ms": rep.parse_ms, "build_ms": rep.build_ms,
            "total_ms": rep.total_ms, "device_decoded": rep.device_decoded, "host_threads": rep.host_threads,
            "bytes": rep.bytes, "GB_per_s": rep.bytes / (wall * 1e-3) / 1e9, "vertices": nv, "faces": nf}


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2,3")
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "load_bench.json"))
    ap.add_argument("--reference", action="store_true", help="also time the reference loader on config 2")
    args = ap.parse_args()
    out = {"cores": os.cpu_count(), "runs": []}
    tmp = tempfile.mkdtemp(prefix="gh_load_")
    for k in [int(x) for x in args.configs.split(",")]:
        w = meshgen.config(k)
        mesh = g.build_mesh(w.positions, w.faces)
        for fmt, ext in ((g.MeshFormat.PLY, "ply"), (g.MeshFormat.OBJ, "obj")):
            path = os.path.join(tmp, f"c{k}.{ext}")
            t0 = time.perf_counter()
            g.save_mesh(path, mesh)
            save_ms = (time.perf_counter() - t0) * 1e3
            r = time_load(path)
            r.update({"config": k, "format": ext, "save_ms": save_ms})
            out["runs"].append(r)
            print(json.dumps(r), flush=True)
            if args.reference and k == 2:
                from oracle.oracle import Oracle
                o = Oracle("reference")
                data = open(path, "rb").read()
                t0 = time.perf_counter()
                om = o.load_mesh(data, int(fmt))
                ref_load = (time.perf_counter() - t0) * 1e3
                del om
                t0 = time.perf_counter()
                om = o.build_mesh(w.positions, w.faces)
                ref_build = (time.perf_counter() - t0) * 1e3
                del om
                rr = {"config": k, "format": ext, "impl": "reference", "load_plus_build_ms": ref_load,
                      "build_only_ms": ref_build, "parse_ms": ref_load - ref_build, "threads": 1}
                out["runs"].append(rr)
                print(json.dumps(rr), flush=True)
            os.unlink(path)
        del mesh
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
