"""CPU-side checks of the boundary: libexpd.so loads (no GPU needed to dlopen it), it
exports every symbol include/expd.h declares, the Python binding names match, and the
product package never reaches into oracle/ (the oracle is test infrastructure)."""
from __future__ import annotations

import ast
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "expd.h")
PKG = os.path.join(ROOT, "paper_2603_04350_b200")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(expd_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2603_04350_b200 import build

    return build.build()


def test_library_exports_every_declared_symbol(libpath):
    lib = ctypes.CDLL(libpath)
    missing = [f for f in header_functions() if not hasattr(lib, f)]
    assert not missing, missing


def test_nm_shows_c_linkage(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True).stdout
    syms = {l.split()[-1] for l in out.splitlines() if l.strip()}
    for f in header_functions():
        assert f in syms, f  # unmangled: extern "C"


def test_binding_covers_header():
    from paper_2603_04350_b200.expd import EXPORTS

    assert sorted(EXPORTS) == header_functions()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] in ("oracle", "synth") for a in node.names), p
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] not in ("oracle", "synth"), p
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(p).read().lower(), p


def test_plan_requires_cuda_or_fails_loudly():
    import torch

    from paper_2603_04350_b200 import Plan, Problem

    if torch.cuda.is_available():
        pytest.skip("GPU present: covered by the gpu tests")
    with pytest.raises(RuntimeError):
        Plan(Problem(1, 7, 1.0, 1.0, 0.1, 8, 1e-2))
