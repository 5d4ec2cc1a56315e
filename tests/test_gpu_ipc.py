"""Two processes, one GPU: the multi-process partition path through CUDA IPC.

A child process owns part 1 of a 2-part partition (sector slices or BFS
bands) and exports its buffers (gh_band_export). This process builds part 0,
adopts the child's part 1 buffers (gh_band_adopt: cudaIpcOpenMemHandle) and
runs both parts in one cooperative launch (gh_band_launch_group) with
system-scope releases and polls — the peer stores and counter updates of the
multi-GPU kernel, landing in the other process's allocation. Two kernels that
wait on each other are never run as separate processes on one GPU (Xid 109,
B200_PROFILING.md); one launch drives both parts instead. Checks: u bitwise
equal to gs_diffuse, and the child reads its own rows back from its own
memory, bitwise equal too.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("partition", ["slices", "bands"])
def test_two_process_ipc_partition_bitwise(gpu, tmp_path, partition):
    from paper_1812_06060_b200 import bands, meshgen
    gh = gpu
    sweeps = 37
    P, F, S = meshgen.torus(96, 48, 1.0, 0.3, 3e-4, 5, 2)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, S)
    t = gh.diffusion_time(mesh, 1.0)
    want = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=sweeps))
    gh.geoheat.release_cached_memory()
    child = subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "ipc_part.py"), str(tmp_path), partition,
                              "1", "2", str(sweeps)], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    try:
        blob_path = tmp_path / "blob1"
        import time
        t0 = time.time()
        while not blob_path.exists():
            assert child.poll() is None, child.stdout.read()
            assert time.time() - t0 < 180, "child did not export its part"
            time.sleep(0.02)
        p0 = bands.Band(lv, 0, 2, partition=partition)
        p1 = bands.Band(lv, 1, 2, partition=partition)
        p1.adopt(blob_path.read_bytes())
        got = bands.launch_group([p0, p1], t, sweeps)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        (tmp_path / "launched").write_text("1")
        own_path = tmp_path / "own1.npy"
        t0 = time.time()
        while not own_path.exists():
            assert child.poll() is None, child.stdout.read()
            assert time.time() - t0 < 180, "child did not read its rows back"
            time.sleep(0.02)
        u1, mask = np.load(own_path)
        mask = mask.astype(bool)
        assert mask.sum() > 0 and mask.sum() < mask.size
        assert np.array_equal(u1[mask].view(np.uint64), want[mask].view(np.uint64))
        del p1, p0  # unmap the child's buffers before it frees them
        import gc
        gc.collect()
    finally:
        (tmp_path / "launched").write_text("1")  # never leave the child waiting
        (tmp_path / "exit").write_text("1")
        try:
            out, _ = child.communicate(timeout=120)
        except subprocess.TimeoutExpired:
            child.kill()
            raise
    assert child.returncode == 0, out


def test_launch_group_local_parts_bitwise(gpu):
    """launch_group with every part local equals gs_diffuse (slices and bands, 1-4 parts)."""
    from paper_1812_06060_b200 import bands, meshgen
    gh = gpu
    P, F, S = meshgen.torus(80, 40, 1.0, 0.3, 3e-4, 9, 3)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, S)
    t = gh.diffusion_time(mesh, 1.0)
    want = gh.gs_diffuse(mesh, lv, t, gh.DiffusionConfig(sweeps=21))
    for partition in ("slices", "bands"):
        for n in (1, 2, 3, 4):
            parts = [bands.Band(lv, r, n, partition=partition) for r in range(n)]
            got = bands.launch_group(parts, t, 21)
            assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (partition, n)
            if n > 1:
                with pytest.raises(ValueError):
                    bands.launch_group(parts[::-1], t, 21)
