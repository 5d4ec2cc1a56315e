"""bench.py keeps the driver's JSON-line contract (keys, units, types).

CPU: the reference arm (`--impl reference`) on config 1 — the compiled
reference's gs_diffuse on the host cores. GPU: our arm on config 2 with fewer
sweeps (the metric, roofline, e2e, clocks and launch-count keys)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "1", "--steps", "2", "--warmup", "1", "--cpu-sample-sweeps", "50"],
             600)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "vertex-updates/s"
    assert d["metric"] == "vertex-updates/s per solver sweep" and d["higher_is_better"] is True
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("C1 ")


@pytest.mark.gpu
def test_our_arm_line():
    d = _run(["--config", "2", "--steps", "2", "--warmup", "3", "--sweeps", "100", "--e2e-steps", "1",
              "--no-cpu-baseline"], 900)
    assert BASE_KEYS <= set(d)
    assert d["value"] > 1e9 and d["dtype"] == "f64" and d["n_gpus"] == 1
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and r["achieved"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_recorded_traffic_matches_default_workload():
    """roofline.traffic: the committed ncu capture (profiles/diffusion_traffic.json) is found
    for the default bench workload (config 3, face) whatever the sweep / ADMM counts in its label."""
    import importlib.util
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    t, src = b.recorded_traffic("C3 torus4096x2048 face, 1000 sweeps, 10 ADMM iters", 1000)
    assert t is not None and src
    assert 0.5 * 838860800000 < t < 1.2 * 838860800000  # DRAM bytes per 1000-sweep launch vs algorithmic
    assert b.recorded_traffic("C2 grid1025 face, 1000 sweeps, 10 ADMM iters", 1000) == (None, None)
