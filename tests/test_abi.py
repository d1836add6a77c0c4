"""CPU-side checks of the boundary: libmsb.so builds, loads, and exports every
symbol declared in include/msb.h; the binding declares every one of them; the
product package never imports the oracle; no CPU fallback exists."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2001_01624_b200")


def header_symbols():
    src = open(os.path.join(ROOT, "include", "msb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(msb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_all_header_symbols():
    from paper_2001_01624_b200 import build
    lib_path = build.build()
    import ctypes
    lib = ctypes.CDLL(lib_path)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_declares_all_symbols():
    from paper_2001_01624_b200 import _lib
    assert set(header_symbols()) == set(_lib.SIGNATURES)
    lib = _lib.load()
    assert lib.msb_version().decode().startswith("libmsb")


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.startswith("oracle") for a in node.names), f
                    if isinstance(node, ast.ImportFrom):
                        assert not (node.module or "").startswith("oracle"), f


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2001_01624_b200 import Context, MsbError
    with pytest.raises(MsbError):
        Context(0)


def test_sources_target_sm100a():
    from paper_2001_01624_b200 import build
    assert "arch=compute_100a,code=sm_100a" in " ".join(build.ARCH)
