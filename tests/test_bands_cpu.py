"""Multi-GPU partitions, host side (CPU, gloo): the band plan, and the band and
sector-slice decompositions of the pipelined diffusion run as world_size 2-4
process groups exchanging halos, bit-identical to the reference's gs_diffuse."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLDEN, ROOT
from paper_1812_06060_b200 import bands


def test_plan_matches_native_and_balances():
    rng = np.random.default_rng(5)
    for _ in range(50):
        nlev = int(rng.integers(1, 60))
        sizes = rng.integers(1, 400, nlev)
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        for n in range(1, min(nlev, 9) + 1):
            cut = bands.plan_bands(off, n)
            assert cut == bands.plan_bands_native(off, n)
            assert cut[0] == 0 and cut[-1] == nlev and all(a < b for a, b in zip(cut, cut[1:]))
    with pytest.raises(ValueError):
        bands.plan_bands([0, 5], 2)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, queue, partition="bands"):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from band_sim import run_band, run_slice
    from oracle.oracle import Oracle
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    o = Oracle("port")
    mesh = o.build_mesh(g["positions"], g["faces"])
    lv = mesh.bfs(g["sources"])
    arrays = {k: mesh.array(k) for k in ("vv_offset", "vv_index", "vv_weight", "vertex_area", "vertex_weight_sum")}
    levels = dict(level_of_vertex=lv.level_of_vertex, order=lv.order, offsets=lv.offsets)
    if partition == "slices":
        u = run_slice(rank, world, arrays, levels, float(g["t"]), int(g["sweeps"]))
    else:
        plan = bands.plan_bands(lv.offsets, world)
        u = run_band(rank, world, arrays, levels, float(g["t"]), int(g["sweeps"]), plan)
    if rank == 0:
        queue.put((u, g["u"]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [(2, "hex_disk12_two_sources"), (3, "icosphere3"), (2, "two_disjoint_triangles"),
                                        (3, "torus60x30_three_sources")])
def test_band_decomposition_gloo(world, case):
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    if len(g["offsets"]) - 1 < world or int(g["sweeps"]) == 0:
        pytest.skip("fewer levels than ranks")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    u, want = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(u.view(np.uint64), want.view(np.uint64))


@pytest.mark.parametrize("world,case", [(2, "hex_disk12_two_sources"), (3, "icosphere3"), (2, "two_disjoint_triangles"),
                                        (3, "torus60x30_three_sources"), (4, "grid64x40_two_sources")])
def test_slice_decomposition_gloo(world, case):
    """Sector slices (every rank 1/N of every ring, ghost rows exchanged each
    step) as world_size 2-4 gloo process groups: bit-identical to gs_diffuse."""
    g = np.load(os.path.join(GOLDEN, case + ".npz"))
    if int(g["sweeps"]) == 0:
        pytest.skip("no sweeps")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q, "slices")) for r in range(world)]
    for p in procs:
        p.start()
    u, want = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(u.view(np.uint64), want.view(np.uint64))
