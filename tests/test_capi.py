"""The product library loads on CPU and exports every symbol include/plbm_gpu.h
declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from paper_1510_03560_b200 import build, capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols(header):
    text = open(os.path.join(REPO, "include", header)).read()
    return sorted(set(re.findall(r"\b(plbm_gpu_\w+)\s*\(", text)))


def test_header_declares_the_step_loop_boundary():
    syms = declared_symbols("plbm_gpu.h")
    for s in ("plbm_gpu_create", "plbm_gpu_step", "plbm_gpu_read_tile", "plbm_gpu_counters",
              "plbm_gpu_creation_log", "plbm_gpu_destroy"):
        assert s in syms


def test_library_exports_every_declared_symbol():
    build.build_gpu()
    lib = ctypes.CDLL(capi.GPU_LIB)
    missing = [s for s in declared_symbols("plbm_gpu.h") if not hasattr(lib, s)]
    assert not missing, missing


def test_library_is_sm100a_only():
    import subprocess
    build.build_gpu()
    out = subprocess.run(["cuobjdump", "--list-elf", capi.GPU_LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)
