"""Experiment: the diffusion's sweep-group schedule.

For each config, times the 1000-sweep solve with the plain pipeline and with
sweep groups of K sweeps (GH_SWEEP_GROUP=K) under each L2 policy of the CSR
stream (GH_STREAM_L2=0 evict_first, 1 evict_last, 2 evict_normal), and checks
that every variant's u is bit-identical to the plain pipeline's.

    python tools/sweep_groups.py [--configs 3,2] [--groups 16,32,64,128] [--policies 0,1,2] [--reps 3]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import meshgen  # noqa: E402


def solve(mesh, lv, t, sweeps, reps, env):
    for k in ("GH_SWEEP_GROUP", "GH_SWEEP_PERIOD", "GH_STREAM_L2"):
        os.environ.pop(k, None)
    os.environ.update(env)
    ms = []
    u = None
    for _ in range(reps + 1):
        rep = gh.SolverReport()
        u = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps), rep)
        ms.append(rep.device_ms)
    return u, ms[1:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,2")
    ap.add_argument("--groups", default="16,32,64,128")
    ap.add_argument("--policies", default="0,2")
    ap.add_argument("--periods", default="0")
    ap.add_argument("--sweeps", type=int, default=1000)
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    for k in [int(x) for x in a.configs.split(",")]:
        w = meshgen.config(k)
        mesh = gh.build_mesh(w.positions, w.faces)
        lv = gh.bfs_levels(mesh, w.sources)
        t = w.t if w.t is not None else gh.diffusion_time(mesh, w.m)
        reach = mesh.vertex_count() - lv.unreachable_count
        base, ms = solve(mesh, lv, t, a.sweeps, a.reps, {})
        rows = [{"config": k, "group": None, "policy": "auto", "ms": ms}]
        print(json.dumps(dict(rows[-1], gvus=reach * a.sweeps / np.median(ms) / 1e6, levels=lv.level_count())),
              flush=True)
        for g in [int(x) for x in a.groups.split(",")]:
            for p in [int(x) for x in a.policies.split(",")]:
                for per in [int(x) for x in a.periods.split(",")]:
                    env = {"GH_SWEEP_GROUP": str(g), "GH_STREAM_L2": str(p)}
                    if per:
                        env["GH_SWEEP_PERIOD"] = str(per)
                    u, ms = solve(mesh, lv, t, a.sweeps, a.reps, env)
                    same = bool(np.array_equal(u.view(np.uint64), base.view(np.uint64)))
                    print(json.dumps({"config": k, "group": g, "policy": p, "period": per, "ms": ms,
                                      "gvus": reach * a.sweeps / np.median(ms) / 1e6, "bitwise": same}), flush=True)


if __name__ == "__main__":
    main()
