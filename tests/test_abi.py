"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads, and
exports every symbol include/lobster.h declares.  No compute call (no GPU)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "lobster.h")).read()
    return sorted(set(re.findall(r"\b(lobster_[a-z_]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2503_21937_b200 import build
    return build()


def test_header_declares_the_four_calls():
    d = _declared()
    for name in ("lobster_program_load", "lobster_facts_push", "lobster_run", "lobster_output_get"):
        assert name in d


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(lobster_\w+)", out))
    missing = [s for s in _declared() if s not in exported]
    assert not missing, missing
    L = ctypes.CDLL(lib_path)
    for s in _declared():
        assert getattr(L, s) is not None


def test_python_binding_names_match_header(lib_path):
    from paper_2503_21937_b200 import _lib
    assert sorted(_lib.EXPORTS) == _declared()
    L = _lib.load()
    assert L.lobster_create is not None


def test_kernels_are_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_fails_loudly(lib_path):
    """On a host without a CUDA device the engine must not fall back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2503_21937_b200 import Engine, LobsterError, UNIT
    with pytest.raises(LobsterError):
        Engine("type e(x: i32)\nrel r(x) :- e(x).", UNIT)


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2503_21937_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".hpp", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "import oracle" not in txt and "liboracle" not in txt and "oracle.cpp" not in txt, f
