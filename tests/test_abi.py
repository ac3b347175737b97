"""CPU checks of the boundary: the C-ABI library builds, loads, and exports
every symbol include/*.h declares (no compute calls without a GPU)."""
import ctypes
import glob
import os
import re

import pytest

import paper_2001_07104_b200 as rfg
from paper_2001_07104_b200 import build as rfbuild

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        for m in re.finditer(r"RF_API\s+[\w\s\*]+?\b(rf_\w+)\s*\(", open(h).read()):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def libpath():
    return rfbuild.build()


def test_header_matches_binding():
    assert declared_symbols() == set(rfg.ABI_SYMBOLS)


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_binding_loads_without_gpu(libpath):
    L = rfg.lib()
    p = rfg.params(ntree=7, seed=3)
    assert p.struct_size == ctypes.sizeof(rfg.Params) and p.ntree == 7 and p.min_samples_split == 2
    assert p.max_depth == -1 and p.bootstrap == 1
    assert isinstance(L.rf_last_error(), bytes)


def test_no_oracle_imports_in_product():
    pkg = os.path.join(ROOT, "paper_2001_07104_b200")
    for f in glob.glob(os.path.join(pkg, "**", "*"), recursive=True):
        if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
            src = open(f).read()
            assert "oracle" not in re.sub(r"(#|//).*", "", src).lower() or f.endswith("build.py"), f


def test_sm100a_cubin(libpath):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", libpath], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
