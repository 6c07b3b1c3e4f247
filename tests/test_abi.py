"""CPU-side checks of the C-ABI boundary: the shared library loads without a GPU
and exports every symbol include/orca_b200.h declares; the Python mirror of the
structs matches the header; the product refuses to run without CUDA instead of
falling back to a CPU path."""

import ctypes as C
import os
import re

import pytest

from helpers import ROOT
from paper_2008_11578_b200 import _lib

HEADER = os.path.join(ROOT, "include", "orca_b200.h")


def header_symbols():
    src = open(HEADER).read()
    return re.findall(r"^ORCA_API\s+[\w\s\*]+?\b(orca_\w+)\s*\(", src, flags=re.M)


def test_header_and_binding_agree():
    syms = header_symbols()
    assert len(syms) >= 25
    assert sorted(syms) == sorted(_lib.SYMBOLS)


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)      # loading must not need a GPU
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.orca_abi_version() == 2


def test_struct_layouts_match_header():
    # orca_params: 8 doubles + 4 int32; orca_info: 5 int64 + double + 2 int32 + double + 3 int64
    assert C.sizeof(_lib.OrcaParams) == 8 * 8 + 4 * 4
    assert C.sizeof(_lib.OrcaInfo) == 5 * 8 + 8 + 2 * 4 + 8 + 3 * 8
    src = open(HEADER).read()
    assert "#define ORCA_N_STAGES 6" in src and _lib.ORCA_N_STAGES == 6
    assert "ORCA_F32 = 0, ORCA_F64 = 1, ORCA_MIXED = 2, ORCA_CERT32 = 3" in src


def test_no_cpu_fallback_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2008_11578_b200 import Simulation
    from paper_2008_11578_b200.synth import plaza_crowd
    st, cfg = plaza_crowd(8, 0)
    with pytest.raises(_lib.OrcaError) as ei:
        Simulation(cfg, capacity=8)
    assert ei.value.code == -2          # ORCA_ECUDA: fails loudly, no host path
    from paper_2008_11578_b200 import step
    with pytest.raises(_lib.OrcaError):
        step(st, cfg)


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2008_11578_b200")
    for dirpath, _dirs, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, flags=re.M), f
                assert "liborca_oracle" not in text and "orca_oracle" not in text, f
    # outside the package only tests/, bench.py (CPU legs) and __graft_entry__.py (smoke, build)
    # may touch oracle/
    for dirpath, dirs, files in os.walk(ROOT):
        dirs[:] = [d for d in dirs if d not in (".git", "tests", "oracle", "gpurun_out", "__pycache__",
                                               "paper_2008_11578_b200", "variants", ".pytest_cache")]
        for f in files:
            if f.endswith(".py") and not (dirpath == ROOT and f in ("bench.py", "__graft_entry__.py")):
                text = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", text, flags=re.M), os.path.join(dirpath, f)
