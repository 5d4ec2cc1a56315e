"""TEST INFRASTRUCTURE: a numpy restatement of one BFS band of the multi-GPU
diffusion schedule, run one process per band over gloo.

Each rank owns levels [lb, lb') of the plan, keeps both sweep-parity buffers
for its own levels plus ghost copies of levels lb-1 and lb', runs the
pipelined steps tau = L + 2s for its own levels only, and after every step
sends its boundary levels (both parity buffers) to the neighbours, which
overwrite their ghosts. The per-row arithmetic is the reference's
(diffusion.hpp:74-83, row order kept, no FMA), so the gathered u must equal
gs_diffuse bit for bit. This checks the host-side decomposition (plan, ghost
levels, parity buffers, step ranges, halo direction) on CPU.
"""
import numpy as np
import torch
import torch.distributed as dist


def run_band(rank, world, mesh_arrays, levels, t, sweeps, plan):
    off = mesh_arrays["vv_offset"]
    idx = mesh_arrays["vv_index"]
    w = mesh_arrays["vv_weight"]
    va = mesh_arrays["vertex_area"]
    ws = mesh_arrays["vertex_weight_sum"]
    level_of = levels["level_of_vertex"]
    order, loff = levels["order"], levels["offsets"]
    nlev = len(loff) - 1
    V = len(level_of)
    lb, le = plan[rank], plan[rank + 1]
    u0 = (level_of == 0).astype(np.float64)
    buf = [u0.copy(), u0.copy()]  # full-size per rank; only own + ghost levels are ever read
    ring = [order[loff[L]:loff[L + 1]] for L in range(nlev)]

    def update_level(L, s):
        rows = ring[L]
        cur, prev = buf[s & 1], buf[(s & 1) ^ 1]
        deg = off[rows + 1] - off[rows]
        K = int(deg.max()) if rows.size else 0
        num = np.zeros(rows.size)
        for k in range(K):  # sequential row sums in the reference's neighbour order
            has = k < deg
            a = off[rows] + np.minimum(k, deg - 1)
            nb = idx[a]
            val = np.where(level_of[nb] == L - 1, cur[nb], prev[nb])
            num = np.where(has, num + w[a] * val, num)
        den = va[rows] + t * ws[rows]
        cur[rows] = ((L == 0) * 1.0 + t * num) / den

    def exchange():
        reqs, recvs = [], []
        for nbr, send_level, recv_level in ((rank - 1, lb, lb - 1), (rank + 1, le - 1, le)):
            if 0 <= nbr < world:
                out = torch.from_numpy(np.concatenate([buf[0][ring[send_level]], buf[1][ring[send_level]]]))
                inc = torch.empty(2 * ring[recv_level].size, dtype=torch.float64)
                reqs.append(dist.isend(out, nbr))
                reqs.append(dist.irecv(inc, nbr))
                recvs.append((recv_level, inc))
        for r in reqs:
            r.wait()
        for L, inc in recvs:
            n = ring[L].size
            buf[0][ring[L]] = inc[:n].numpy()
            buf[1][ring[L]] = inc[n:].numpy()

    nsteps = (nlev - 1) + 2 * (sweeps - 1) + 1
    for tau in range(nsteps):
        for L in range(lb, le):
            if (tau - L) % 2 == 0 and 0 <= (tau - L) // 2 < sweeps:
                update_level(L, (tau - L) // 2)
        exchange()
    result = buf[(sweeps - 1) & 1]
    mine = (level_of >= lb) & (level_of < le)
    part = torch.from_numpy(np.where(mine, result, 0.0))
    dist.all_reduce(part)
    u = part.numpy()
    u[level_of < 0] = u0[level_of < 0]
    return u


def slice_owner(levels, nslices):
    """Slice of every vertex (-1 unreachable): position p of n in its ring -> p * N // n
    (gh_band.cu k_slice_owner, with the BFS ring order as the layout order)."""
    order, loff = levels["order"], levels["offsets"]
    owner = np.full(len(levels["level_of_vertex"]), -1, np.int64)
    for L in range(len(loff) - 1):
        a, b = int(loff[L]), int(loff[L + 1])
        owner[order[a:b]] = (np.arange(b - a, dtype=np.int64) * nslices) // (b - a)
    return owner


def run_slice(rank, world, mesh_arrays, levels, t, sweeps):
    """One sector slice of the pipelined diffusion: this rank
    updates its 1/N of every ring at every step; after every step it sends the
    rows each other rank ghosts (foreign neighbours of that rank's rows) to it,
    both parity buffers. The gathered own rows must equal gs_diffuse bit for bit."""
    off = mesh_arrays["vv_offset"]
    idx = mesh_arrays["vv_index"]
    w = mesh_arrays["vv_weight"]
    va = mesh_arrays["vertex_area"]
    ws = mesh_arrays["vertex_weight_sum"]
    level_of = levels["level_of_vertex"]
    order, loff = levels["order"], levels["offsets"]
    nlev = len(loff) - 1
    owner = slice_owner(levels, world)
    u0 = (level_of == 0).astype(np.float64)
    buf = [u0.copy(), u0.copy()]
    ring = [order[loff[L]:loff[L + 1]] for L in range(nlev)]
    mine = [r[owner[r] == rank] for r in ring]
    # ghosts of slice d: foreign neighbours of its rows; export[d] = this rank's rows d ghosts
    reach = np.flatnonzero(level_of >= 0)
    src = np.repeat(reach, off[reach + 1] - off[reach])
    nbr = idx[np.concatenate([np.arange(off[v], off[v + 1]) for v in reach])] if reach.size else np.zeros(0, int)
    export = {}
    for d in range(world):
        if d == rank:
            continue
        sel = (owner[src] == d) & (owner[nbr] == rank)
        export[d] = np.unique(nbr[sel])
    imports = {}
    for q in range(world):
        if q == rank:
            continue
        sel = (owner[src] == rank) & (owner[nbr] == q)
        imports[q] = np.unique(nbr[sel])

    def update(rows, L, s):
        cur, prev = buf[s & 1], buf[(s & 1) ^ 1]
        deg = off[rows + 1] - off[rows]
        K = int(deg.max()) if rows.size else 0
        num = np.zeros(rows.size)
        for k in range(K):  # sequential row sums in the reference's neighbour order
            has = k < deg
            a = off[rows] + np.minimum(k, deg - 1)
            nb = idx[a]
            val = np.where(level_of[nb] == L - 1, cur[nb], prev[nb])
            num = np.where(has, num + w[a] * val, num)
        cur[rows] = ((L == 0) * 1.0 + t * num) / (va[rows] + t * ws[rows])

    def exchange():
        reqs, recvs = [], []
        for d, rows in export.items():
            reqs.append(dist.isend(torch.from_numpy(np.concatenate([buf[0][rows], buf[1][rows]])), d))
        for q, rows in imports.items():
            inc = torch.empty(2 * rows.size, dtype=torch.float64)
            reqs.append(dist.irecv(inc, q))
            recvs.append((rows, inc))
        for r in reqs:
            r.wait()
        for rows, inc in recvs:
            buf[0][rows] = inc[:rows.size].numpy()
            buf[1][rows] = inc[rows.size:].numpy()

    nsteps = (nlev - 1) + 2 * (sweeps - 1) + 1
    for tau in range(nsteps):
        for L in range(nlev):
            if (tau - L) % 2 == 0 and 0 <= (tau - L) // 2 < sweeps and mine[L].size:
                update(mine[L], L, (tau - L) // 2)
        exchange()
    result = buf[(sweeps - 1) & 1]
    part = torch.from_numpy(np.where(owner == rank, result, 0.0))
    dist.all_reduce(part)
    u = part.numpy()
    u[level_of < 0] = u0[level_of < 0]
    return u
