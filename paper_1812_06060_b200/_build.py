"""Build recipes for the in-tree native libraries (run by __graft_entry__.build()).

  lib/libgeoheat_b200.so   the CUDA path: csrc/*.cu for sm_100a, fp64 with
                           FMA contraction off (-fmad=false) so element values
                           match the reference bit for bit.
  lib/libgh_meshgen.so     host C mesh generators for the BASELINE configs (workloads/meshgen.c).

The libraries are built in place (not pip-installed) so they travel with the
repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
CUDA_LIB = os.path.join(LIBDIR, "libgeoheat_b200.so")
MESHGEN_LIB = os.path.join(LIBDIR, "libgh_meshgen.so")
# the seeded BASELINE workloads (not the solver path): shared with the CPU
# reference arm, which builds its own copy under oracle/_ref/
MESHGEN_SRC = os.path.join(ROOT, "workloads", "meshgen.c")
CLI_BIN = os.path.join(LIBDIR, "geoheat_b200")
CLI_SRC = os.path.join(PKG, "cli", "geoheat_cli.cpp")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-fmad=false", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
                     "-Xptxas", "-v", "-I", os.path.join(ROOT, "include")]

HOST_FLAGS = ["-std=c++17", "-O3", "-fPIC", "-g1", "-Wall", "-pthread", "-ffp-contract=off"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: str, sources) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(s) <= t for s in sources)


def build_meshgen(force: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    src = MESHGEN_SRC
    if force or not _newer(MESHGEN_LIB, [src]):
        tmp = MESHGEN_LIB + ".tmp"
        subprocess.run(["gcc", "-std=gnu11", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-o", tmp, src, "-lm"],
                       check=True)
        os.replace(tmp, MESHGEN_LIB)
    return MESHGEN_LIB


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(LIBDIR, exist_ok=True)
    sources = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    host_sources = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    headers = (sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + sorted(glob.glob(os.path.join(CSRC, "*.hpp"))) +
               [os.path.join(ROOT, "include", "geoheat_b200.h")])
    sources_all = sources + host_sources
    if not force and _newer(CUDA_LIB, sources_all + headers):
        return CUDA_LIB
    nvcc = _nvcc()
    objdir = os.path.join(LIBDIR, "obj")
    os.makedirs(objdir, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if src.endswith(".cpp"):  # host-only code (mesh I/O): the host compiler directly
            cmd = ["g++", *HOST_FLAGS, "-c", src, "-o", obj]
        else:
            cmd = [nvcc, *NVCC_FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(r.stderr)
        return obj

    with cf.ThreadPoolExecutor(max_workers=min(8, len(sources))) as ex:
        objs = list(ex.map(compile_one, sources_all))
    tmp = CUDA_LIB + ".tmp"
    r = subprocess.run([nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-lpthread"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, CUDA_LIB)
    if verbose:
        for o in objs:
            print(open(o + ".ptxas.txt").read())
    return CUDA_LIB


def build_cli(force: bool = False) -> str:
    """The reference CLI (tools/geoheat.cpp) on the C ABI: lib/geoheat_b200."""
    lib = build_cuda()
    header = os.path.join(ROOT, "include", "geoheat_b200.h")
    if force or not _newer(CLI_BIN, [CLI_SRC, header, lib]):
        tmp = CLI_BIN + ".tmp"
        r = subprocess.run(["g++", "-std=c++17", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-o", tmp, CLI_SRC,
                            "-L", LIBDIR, "-lgeoheat_b200", "-Wl,-rpath,$ORIGIN", "-pthread"],
                           capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"CLI build failed:\n{r.stderr}")
        os.replace(tmp, CLI_BIN)
    return CLI_BIN


REF = "/root/reference/proj"


def build_test_programs(force: bool = False) -> list:
    """Test infrastructure, not product: the C++ programs the GPU tests run.

    lib/wrapper_parity       the reference's run_pipelines chain on include/geoheat_b200.hpp
    lib/dropin_run_pipeline  that chain on the reference's own functions and on
                             geoheat::b200 with the reference's types (needs the
                             reference headers, so only where /root/reference exists)
    """
    lib = build_cuda()
    meshgen = build_meshgen()
    inc = os.path.join(ROOT, "include")
    built = []
    jobs = [("wrapper_parity", ["g++", "-std=c++20", "-O2", "-Wall", "-I", inc], ["-lgh_meshgen"], True)]
    if os.path.isdir(os.path.join(REF, "include", "geoheat")):
        jobs.append(("dropin_run_pipeline",
                     ["g++", "-std=gnu++20", "-O2", "-fopenmp", "-ffp-contract=off", "-I",
                      os.path.join(ROOT, "oracle", "eigen_shim"), "-I", REF + "/include", "-I", REF + "/tests", "-I", inc],
                     [], True))
    for name, head, extra, _ in jobs:
        src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
        exe = os.path.join(LIBDIR, name)
        if force or not _newer(exe, [src, lib, meshgen, os.path.join(inc, "geoheat_b200.hpp")]):
            r = subprocess.run(head + [src, "-o", exe + ".tmp", "-L", LIBDIR, "-lgeoheat_b200", *extra,
                                       "-Wl,-rpath,$ORIGIN"], capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"{name} build failed:\n{r.stderr[-3000:]}")
            os.replace(exe + ".tmp", exe)
        built.append(exe)
    return built


def build_all(force: bool = False) -> None:
    build_meshgen(force)
    build_cuda(force)
    build_cli(force)
    build_test_programs(force)


if __name__ == "__main__":
    import sys
    build_all(force="--force" in sys.argv)
    print(CUDA_LIB)
