"""The C-ABI library builds for sm_100a, loads and exports every symbol that
include/lyap_ir.h declares (no compute calls: runs without a GPU)."""
import ctypes
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "lyap_ir.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(lyap_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_header_symbols():
    import paper_2510_02126_b200 as G
    import importlib
    B = importlib.import_module("paper_2510_02126_b200.build")
    B.build()
    lib = ctypes.CDLL(G.library_path())
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(lib, s), s
    assert set(G.SYMBOLS) <= set(syms)


def test_library_is_sm100a():
    import paper_2510_02126_b200 as G
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", G.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_path_has_no_oracle_dependency():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2510_02126_b200")
    for dp, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dp, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "oracle.h" not in src and "liblyaporacle" not in src, f


def test_no_cuda_device_fails_loudly():
    import torch
    import pytest
    import paper_2510_02126_b200 as G
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(G.LyapError):
        G.Solver(8)
