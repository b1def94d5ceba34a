"""Host-side checks of the C-ABI library that need no GPU: it builds for sm_100a, loads, exports
every symbol include/specedge.h declares, contains tcgen05/TMA code, and the product package is
independent of the oracle."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2505_17052_b200 import build
    return build.build()


def _header_functions():
    src = open(os.path.join(ROOT, "include", "specedge.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(specedge_\w+)\s*\(", src)))


def test_header_declares_and_library_exports_every_symbol(libpath):
    from paper_2505_17052_b200 import _lib
    declared = _header_functions()
    assert declared == sorted(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\b(specedge_\w+)\b", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    lib = ctypes.CDLL(libpath)
    for f in declared:
        assert hasattr(lib, f)


def test_library_is_sm100a_with_tcgen05_and_tma(libpath):
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", libpath], capture_output=True, text=True,
                          check=True).stdout
    assert "sm_100a" in subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", libpath], capture_output=True,
                                       text=True).stdout
    for mnemonic in ("UTCHMMA", "UTMALDG", "LDTM"):
        assert mnemonic in sass, mnemonic


def test_api_errors_without_device(libpath):
    """Host-detected API misuse returns negative codes before any launch."""
    from paper_2505_17052_b200 import _lib
    lib = _lib.load(libpath)
    out = ctypes.c_void_p()
    assert lib.specedge_model_create(None, 1, 0, ctypes.byref(out)) == _lib.E_INVALID
    assert lib.specedge_verify_batch(None, None, None, None, None, 0, None) == _lib.E_INVALID
    bad = _lib.ModelConfig(2, 64, 4, 2, 24, 256, 256, 1e-6, 1e4, 128)   # head_dim 24 unsupported
    assert lib.specedge_model_create(ctypes.byref(bad), 1, 0, ctypes.byref(out)) == _lib.E_UNSUPPORTED
    # tensor-parallel shards: rank/size/id checks, divisibility of heads / ffn
    ok = _lib.ModelConfig(2, 512, 8, 2, 128, 1024, 2048, 1e-5, 5e5, 128)
    nid = (ctypes.c_uint8 * 128)()
    create_tp = lib.specedge_model_create_tp
    assert create_tp(ctypes.byref(ok), 1, 0, 2, 2, ctypes.cast(nid, ctypes.c_void_p), ctypes.byref(out)) == _lib.E_INVALID
    assert create_tp(ctypes.byref(ok), 1, 0, 0, 0, None, ctypes.byref(out)) == _lib.E_INVALID
    assert create_tp(ctypes.byref(ok), 1, 0, 0, 4, ctypes.cast(nid, ctypes.c_void_p), ctypes.byref(out)) == \
        _lib.E_UNSUPPORTED   # n_kv = 2 not divisible by 4
    assert lib.specedge_model_tp_info(None, None, None, None, None) == _lib.E_INVALID
    assert lib.specedge_tp_fused_enable(None, 64, None) == _lib.E_INVALID


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2505_17052_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", txt, re.M), f
                assert not re.search(r"#include\s+[<\"].*oracle", txt), f
                assert "importlib" not in txt, f
