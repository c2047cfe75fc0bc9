"""CPU-only checks of the boundary: the C-ABI library builds for sm_100a, loads, and exports every
symbol include/shiftk.h declares; the Python binding mirrors the header; the product package
never imports the oracle (no CPU fallback path exists)."""
import ast
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "shiftk.h")
PKG = os.path.join(ROOT, "paper_2001_08707_b200")


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sk_[a-z_]+)\s*\(", src)))


def test_library_builds_and_exports_header_symbols():
    from paper_2001_08707_b200 import build as b
    lib = b.build()
    assert os.path.exists(lib)
    L = ctypes.CDLL(lib)
    fns = header_functions()
    assert len(fns) >= 14
    for name in fns:
        assert hasattr(L, name), name


def test_binding_covers_header():
    from paper_2001_08707_b200 import shiftk
    assert sorted(shiftk.EXPORTS) == header_functions()


def test_version_and_error_strings_without_gpu():
    from paper_2001_08707_b200 import build as b, shiftk
    b.build()
    L = shiftk.load()
    assert b"sm_100a" in L.sk_version()
    assert isinstance(L.sk_last_error(), bytes)
    # null-argument validation happens before any CUDA call
    assert L.sk_init(None, None, None, None) == -1
    assert L.sk_finalize(None) == -5


def test_struct_layouts_match_header():
    from paper_2001_08707_b200 import shiftk
    # sizes fixed by the header's field order (natural alignment, x86-64)
    assert ctypes.sizeof(shiftk.sk_cplx) == 16
    assert ctypes.sizeof(shiftk.sk_operator) == 4 + 4 + 8 + 8 * 4 + 8 * 3 + 4 + 4
    assert ctypes.sizeof(shiftk.sk_params) == 4 + 4 + 8 + 8 + 8 + 4 + 4 + 8 + 8 + 4 + 4 + 8 + 8
    assert ctypes.sizeof(shiftk.sk_dist) == 16 + 16 + 8


def test_sm100a_cubin_inside():
    """The .so carries sm_100a SASS (no PTX JIT path, no other arch)."""
    import subprocess
    from paper_2001_08707_b200 import build as b
    lib = b.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def _imports(path):
    tree = ast.parse(open(path).read())
    mods = set()
    for node in ast.walk(tree):
        if isinstance(node, ast.Import):
            mods |= {a.name.split(".")[0] for a in node.names}
        elif isinstance(node, ast.ImportFrom) and node.module:
            mods.add(node.module.split(".")[0])
    return mods


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                assert "oracle" not in _imports(os.path.join(dirpath, f)), f
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(os.path.join(dirpath, f)).read().lower().replace(
                    "the cpu oracle in oracle/ shares nothing", ""), f


def test_oracle_never_imports_product():
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith(".py"):
            assert "paper_2001_08707_b200" not in _imports(os.path.join(ROOT, "oracle", f))
        if f.endswith(".c"):
            assert "shiftk.h" not in open(os.path.join(ROOT, "oracle", f)).read()
