"""BFS-band sharding of the diffusion across GPUs.

Levels are cut into contiguous bands of about equal row counts
(`plan_bands`, the same integer plan as gh::plan_bands). Band r computes its
own levels [lb, le) and keeps ghost copies of levels lb-1 and le; by the BFS
property those are the only levels its rows touch. The neighbours write the
ghosts directly (peer stores through CUDA IPC mappings + per-level progress
counters) from inside the one dataflow kernel, so no collective runs per step.

Multi-process use (one process per GPU, torch.distributed for the plumbing):

    band = Band(levels, rank, world)
    band.connect_via(dist)            # all_gather of the IPC blobs, then map the neighbours
    band.prepare(t)                   # every rank
    dist.barrier()                    # all counters zeroed before any kernel runs
    u = band.launch(t, sweeps)        # this rank's vertices of u
    dist.barrier()                    # before the next prepare: a neighbour's last
                                      # sweep still writes into our ghost rows and
                                      # counters after our own kernel returned

`gs_diffuse_bands` runs the same schedule with all bands on one GPU in one
launch (the single-GPU emulation used by the tests).

Sector slices (`partition="slices"`) cut every ring instead:
slice r owns positions [ceil(r n / N), ceil((r + 1) n / N)) of each ring of n
vertices, so every rank has work at every pipeline step; the foreign
neighbours of its rows are ghost rows their owners write. Slices connect to
every rank (`connect_all`), bands to their two neighbours.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .geoheat import BfsLevels, SolverReport, TriMesh, _check, _f64, _ptr, gh_solver_report


def plan_bands(offsets: Sequence[int], nbands: int) -> list:
    """Cut levels into nbands contiguous bands of about equal rows; band r owns
    levels [cut[r], cut[r+1]). Mirrors gh::plan_bands (csrc/gh_band.cu)."""
    off = [int(x) for x in offsets]
    nlev = len(off) - 1
    if nbands < 1:
        raise ValueError("plan_bands: need at least one band")
    if nbands > nlev:
        raise ValueError("plan_bands: more bands than BFS levels")
    total = off[nlev]
    cut = [0] * (nbands + 1)
    cut[nbands] = nlev
    L = 0
    for r in range(1, nbands):
        target = total * r // nbands
        while L < nlev and off[L] < target:
            L += 1
        if L > 0 and target - off[L - 1] < off[L] - target:
            L -= 1
        L = max(L, cut[r - 1] + 1)
        L = min(L, nlev - (nbands - r))
        cut[r] = L
    return cut


def plan_bands_native(offsets: Sequence[int], nbands: int) -> list:
    off = np.ascontiguousarray(offsets, dtype=np.int32)
    cut = np.zeros(nbands + 1, np.int32)
    _check(_lib.load().gh_plan_bands(_ptr(off), off.size - 1, int(nbands), _ptr(cut)))
    return cut.tolist()


PARTITIONS = {"bands": 0, "slices": 1}


def gs_diffuse_bands(mesh: TriMesh, levels: BfsLevels, nbands: int, t: float, sweeps: int, initial=None,
                     report: Optional[SolverReport] = None, partition: str = "bands") -> np.ndarray:
    """gs_diffuse split into nbands BFS bands (or sector slices), all on this GPU in one launch."""
    init = None if initial is None else _f64(initial)
    u = np.empty(mesh.vertex_count(), np.float64)
    rep = gh_solver_report()
    _check(mesh._lib.gh_gs_diffuse_partitioned(levels._h, int(nbands), PARTITIONS[partition], float(t), int(sweeps),
                                               _ptr(init), _ptr(u), C.byref(rep)))
    if report is not None:
        report.iterations, report.device_ms, report.kernel_launches = rep.iterations, rep.device_ms, rep.kernel_launches
    return u


def gs_diffuse_slices(mesh: TriMesh, levels: BfsLevels, nslices: int, t: float, sweeps: int, initial=None,
                      report: Optional[SolverReport] = None) -> np.ndarray:
    """gs_diffuse split into nslices sector slices (every slice a 1/N of every ring), one launch."""
    return gs_diffuse_bands(mesh, levels, nslices, t, sweeps, initial, report, partition="slices")


class Band:
    """This process's band of a multi-GPU diffusion (one gh_band handle)."""

    def __init__(self, levels: BfsLevels, rank: int, world: int, partition: str = "bands"):
        self.levels, self.rank, self.world, self.partition = levels, rank, world, partition
        self._lib = levels._lib
        self._h = C.c_void_p()
        _check(self._lib.gh_band_create_partitioned(levels._h, int(rank), int(world), PARTITIONS[partition],
                                                    C.byref(self._h)))
        lb, le, rows = C.c_int32(), C.c_int32(), C.c_int32()
        _check(self._lib.gh_band_info(self._h, C.byref(lb), C.byref(le), C.byref(rows)))
        self.lb, self.le, self.own_rows = lb.value, le.value, rows.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._lib.gh_band_destroy(h)
            self._h = None

    def export(self) -> bytes:
        n = C.c_int32()
        _check(self._lib.gh_band_export(self._h, None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value)
        _check(self._lib.gh_band_export(self._h, buf, n.value, C.byref(n)))
        return buf.raw[:n.value]

    def connect(self, lower: Optional[bytes], upper: Optional[bytes]) -> None:
        _check(self._lib.gh_band_connect(self._h, lower, upper))

    def connect_all(self, blobs) -> None:
        arr = (C.c_char_p * len(blobs))(*[bytes(x) for x in blobs])
        _check(self._lib.gh_band_connect_all(self._h, arr, len(blobs)))

    def connect_via(self, dist) -> None:
        """Exchange IPC blobs with every rank (all_gather_object) and map the two
        neighbours (bands) or every other rank (slices)."""
        blobs = [None] * self.world
        dist.all_gather_object(blobs, self.export())
        if self.partition == "slices":
            self.connect_all(blobs)
        else:
            self.connect(blobs[self.rank - 1] if self.rank > 0 else None,
                         blobs[self.rank + 1] if self.rank + 1 < self.world else None)

    def prepare(self, t: float, initial=None) -> None:
        init = None if initial is None else _f64(initial)
        _check(self._lib.gh_band_prepare(self._h, float(t), _ptr(init)))

    def launch(self, t: float, sweeps: int, report: Optional[SolverReport] = None, copy_out: bool = True):
        u = np.empty(self.levels.mesh.vertex_count(), np.float64) if copy_out else None
        rep = gh_solver_report()
        _check(self._lib.gh_band_launch(self._h, float(t), int(sweeps), _ptr(u), C.byref(rep)))
        if report is not None:
            report.iterations, report.device_ms, report.kernel_launches = rep.iterations, rep.device_ms, \
                rep.kernel_launches
        return u

    def adopt(self, blob: bytes) -> None:
        """Drive another process's copy of this part: map its buffers (its export()) in place of ours."""
        _check(self._lib.gh_band_adopt(self._h, bytes(blob)))

    def download(self, sweeps: int, u: Optional[np.ndarray] = None) -> np.ndarray:
        """This part's own rows of u after `sweeps` sweeps, in vertex order (other entries of u kept, else NaN)."""
        out = np.full(self.levels.mesh.vertex_count(), np.nan) if u is None else np.ascontiguousarray(u, np.float64)
        _check(self._lib.gh_band_download(self._h, int(sweeps), _ptr(out)))
        return out

    def own_mask(self) -> np.ndarray:
        """Vertices whose u this rank computes (its rows of the diffusion layout)."""
        m = np.zeros(self.levels.mesh.vertex_count(), np.uint8)
        _check(self._lib.gh_band_own_mask(self._h, _ptr(m)))
        return m.astype(bool)


def launch_group(parts: Sequence[Band], t: float, sweeps: int, initial=None,
                 report: Optional[SolverReport] = None) -> np.ndarray:
    """Parts 0..n-1 of one partition (some possibly adopted from other processes) in one launch on this GPU."""
    lib = parts[0]._lib
    arr = (C.c_void_p * len(parts))(*[p._h.value for p in parts])
    init = None if initial is None else _f64(initial)
    u = np.empty(parts[0].levels.mesh.vertex_count(), np.float64)
    rep = gh_solver_report()
    _check(lib.gh_band_launch_group(arr, len(parts), float(t), int(sweeps), _ptr(init), _ptr(u), C.byref(rep)))
    if report is not None:
        report.iterations, report.device_ms, report.kernel_launches = rep.iterations, rep.device_ms, rep.kernel_launches
    return u
