"""The C-ABI library builds, loads and exports every symbol include/apo.h
declares (no GPU needed: no compute calls here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "apo.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apo_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2406_18111_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("apo_ingest", "apo_find_repeats", "apo_find_repeats_batched", "apo_suffix_array",
              "apo_candidates", "apo_ctx_create"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(lib):
    import paper_2406_18111_b200 as pkg
    assert set(declared_functions()) <= set(pkg.exported_symbols())


def test_version_and_invalid_args_without_gpu(lib):
    lib.apo_version.restype = ctypes.c_int
    assert lib.apo_version() >= 1
    lib.apo_ctx_create.argtypes = [ctypes.c_int, ctypes.c_void_p]
    assert lib.apo_ctx_create(0, None) == 1          # APO_ERR_INVALID, no device touched
    lib.apo_find_repeats.restype = ctypes.c_int
    assert lib.apo_find_repeats(None, None, 0, 1, None, None, 0, None, 0, None, None) == 1


def test_library_is_sm100a(lib):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          os.path.join(ROOT, "paper_2406_18111_b200", "libapo.so")],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2406_18111_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("no CPU", ""), f


def test_ruler_slices_host_logic(lib):
    """apo_ingest's schedule (apo_ruler_slices, pure host code in libapo) vs
    the oracle's ruler (P:750-755 and R13) for several (C, B), split points
    and start counts; no device needed."""
    import oracle
    from paper_2406_18111_b200.apo import ruler_slices
    assert ruler_slices(0, 4, 1, 8) == [(0, 1), (0, 2), (2, 3), (0, 4)]   # 1, 2, 1, 4
    for C, B in ((1, 8), (250, 5000), (500, 5000), (256, 16384), (3, 7)):
        for k0, n in ((0, 20000), (7, 1), (C * 5 - 1, 2), (12345, 9876)):
            assert ruler_slices(k0, n, C, B) == oracle.ruler_slices(k0, k0 + n, C, B), (C, B, k0, n)
    from paper_2406_18111_b200.apo import ApoError
    with pytest.raises(ApoError):
        ruler_slices(0, 10, 0, 8)
