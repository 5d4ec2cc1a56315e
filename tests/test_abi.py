"""The drop-in boundary (CPU): the C-ABI library loads, exports every symbol
include/geoheat_b200.h declares, the ctypes table matches the header, and with
no GPU the path fails loudly instead of falling back to the CPU."""
import os
import re
import subprocess

import pytest

from conftest import ROOT
from paper_1812_06060_b200 import _build, _lib

HEADER = os.path.join(ROOT, "include", "geoheat_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gh_[a-z0-9_]+)\s*\(", text)))


def test_library_builds_and_loads():
    path = _build.build_cuda()
    assert os.path.exists(path)
    _lib.load()


def test_every_declared_symbol_is_exported():
    names = declared_functions()
    assert len(names) >= 25
    out = subprocess.run(["nm", "-D", "--defined-only", _build.CUDA_LIB], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (gh_[a-z0-9_]+)", out))
    missing = [n for n in names if n not in exported]
    assert not missing, missing


def test_ctypes_table_matches_header():
    assert sorted(n for n, _, _ in _lib.SIGNATURES) == declared_functions()


def test_sm100a_code_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _build.CUDA_LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_field_hash_matches_reference_fnv():
    import numpy as np
    from paper_1812_06060_b200 import geoheat
    assert geoheat.field_hash(np.array([], np.float64)) == 1469598103934665603  # FNV offset basis
    g = np.load(os.path.join(ROOT, "tests", "golden", "icosphere5_config1.npz"))
    assert geoheat.field_hash(g["d_face"]) == 0xcca540701b66bfd5


def _has_gpu():
    from paper_1812_06060_b200 import geoheat
    return geoheat.device_count() > 0


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU error path")
def test_no_gpu_fails_loudly():
    import numpy as np
    from paper_1812_06060_b200 import geoheat
    with pytest.raises(geoheat.GeoheatCudaError, match="no CUDA device"):
        geoheat.build_mesh(np.zeros((3, 3)), np.array([[0, 1, 2]]))


def test_cpp_wrapper_compiles():
    """include/geoheat_b200.hpp (the reference-signature C++ wrapper) builds against the ABI."""
    exes = _build.build_test_programs(force=True)
    assert any(e.endswith("wrapper_parity") for e in exes)


REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.isdir(REF + "/include/geoheat"), reason="needs the reference headers (build container)")
def test_dropin_compiles_against_reference_types():
    """run_pipeline's chain instantiated with the reference's namespace and with
    geoheat::b200 using the reference's own types (GEOHEAT_B200_REFERENCE_TYPES)."""
    exes = _build.build_test_programs()
    assert any(e.endswith("dropin_run_pipeline") for e in exes)
