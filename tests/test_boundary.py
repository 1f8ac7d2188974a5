"""The C-ABI boundary: the in-tree library loads without a GPU, exports exactly what
include/memdet_b200.h declares, and the product never routes through the oracle or a CPU path."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_2503_04424_b200 import _native

HEADER = os.path.join(REPO, "include", "memdet_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(b2d_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    lib = _native.load()
    syms = declared_symbols()
    assert syms, "header declares no functions?"
    for s in syms:
        assert hasattr(lib, s), f"{s} declared in memdet_b200.h but not exported"
    assert set(syms) == set(_native.SIGNATURES), "ctypes signature table out of sync with header"
    assert lib.b2d_version() >= 100


def test_library_is_sm100a():
    so = _native.LIB_PATH
    data = open(so, "rb").read()
    assert b"sm_100a" in data or b"sm_100" in data


def test_product_does_not_import_oracle():
    pkg = os.path.join(REPO, "paper_2503_04424_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b|memdet_oracle|liboracle", text,
                                     re.M), f


def test_no_cpu_fallback_without_gpu():
    lib = _native.load()
    if lib.b2d_device_count() > 0:
        pytest.skip("a GPU is visible")
    import numpy as np

    import paper_2503_04424_b200 as eng

    with pytest.raises(eng.EngineUnavailableError):
        eng.memdet_cholesky(np.eye(4), num_blocks=1)


def test_run_info_struct_matches_header():
    """The ctypes mirror of b2d_run_info / b2d_options must have the header's field order."""
    import re

    text = open(HEADER).read()
    for cname, pyname in (("b2d_run_info", "RunInfoC"), ("b2d_options", "OptionsC"),
                          ("b2d_tilemap", "TileMapC"), ("b2d_tileset", "TileSetC")):
        body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (cname, cname), text, re.S).group(1)
        names = []
        for decl in re.sub(r"/\*.*?\*/", "", body, flags=re.S).split(";"):
            decl = decl.strip()
            if not decl:
                continue
            names += [re.findall(r"(\w+)\s*(?:\[[^\]]*\])?\s*$", n)[0] for n in decl.split(",")]
        assert names == [f[0] for f in getattr(_native, pyname)._fields_], cname
