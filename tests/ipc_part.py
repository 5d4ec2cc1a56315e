"""Child process of tests/test_gpu_ipc.py: owns part `rank` of a 2-part
partition of a small seeded torus, exports its buffers (CUDA IPC blob) and
waits while the parent process drives them; then reads its own rows of u back
from its own allocation and leaves them for the parent to check.

    python tests/ipc_part.py <dir> <partition> <rank> <nparts> <sweeps>
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1812_06060_b200 as gh  # noqa: E402
from paper_1812_06060_b200 import bands, meshgen  # noqa: E402


def wait_for(path, timeout=120.0):
    t0 = time.time()
    while not os.path.exists(path):
        if time.time() - t0 > timeout:
            raise TimeoutError(path)
        time.sleep(0.02)


def main():
    d, partition, rank, nparts, sweeps = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
    P, F, S = meshgen.torus(96, 48, 1.0, 0.3, 3e-4, 5, 2)
    mesh = gh.build_mesh(P, F)
    lv = gh.bfs_levels(mesh, S)
    part = bands.Band(lv, rank, nparts, partition=partition)
    with open(os.path.join(d, f"blob{rank}.tmp"), "wb") as f:
        f.write(part.export())
    os.replace(os.path.join(d, f"blob{rank}.tmp"), os.path.join(d, f"blob{rank}"))
    wait_for(os.path.join(d, "launched"))
    u = part.download(sweeps)
    mask = part.own_mask()
    np.save(os.path.join(d, f"own{rank}.tmp.npy"), np.stack([u, mask.astype(np.float64)]))
    os.replace(os.path.join(d, f"own{rank}.tmp.npy"), os.path.join(d, f"own{rank}.npy"))
    wait_for(os.path.join(d, "exit"))
    del part


if __name__ == "__main__":
    main()
