"""CPU-side checks of the C ABI library: it loads without a GPU and exports every
symbol include/polylla.h declares; host-only calls work; the product path never
imports the oracle and has no CPU fallback."""
import ast
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "polylla.h")).read()
    return sorted(set(re.findall(r"POLYLLA_API\s+[\w\s\*]+?\b(polylla_\w+)\s*\(", src)))


def test_header_symbols_exported():
    import ctypes

    from paper_2403_14723_b200 import polylla as pp
    syms = header_symbols()
    assert len(syms) >= 12
    assert sorted(pp.EXPORTS) == syms
    lib = ctypes.CDLL(pp.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s


def test_workspace_bytes_ex():
    """The bounded layout of polylla_workspace_bytes_ex (NEXT-3): the default is the
    worst case B = 3T with staging; a border bound and no staging shrink it; invalid
    bounds give 0; and index limits are checked before any device access."""
    import ctypes

    from paper_2403_14723_b200 import polylla as pp
    L = pp.lib()
    V, T = 10**6, 2 * 10**6
    assert L.polylla_workspace_bytes_ex(V, T, 3 * T, pp.WS_STAGING, 0) == pp.workspace_bytes(V, T)
    small = L.polylla_workspace_bytes_ex(V, T, 4000, 0, 0)
    assert 0 < small < L.polylla_workspace_bytes_ex(V, T, 4000, pp.WS_STAGING, 0) < pp.workspace_bytes(V, T)
    # origin/twin/next shrink by 3 x 4 B per dropped border slot
    assert L.polylla_workspace_bytes_ex(V, T, 3 * T, 0, 0) - small >= 12 * (3 * T - 4000) - 3 * 256
    assert L.polylla_workspace_bytes_ex(V, T, 3 * T + 1, 0, 0) == 0 and L.polylla_workspace_bytes_ex(V, T, -1, 0, 0) == 0
    h = ctypes.c_void_p()
    fake = ctypes.c_void_p(256)  # aligned, never dereferenced: the checks run first
    # H = 3T + max_border <= 2^32 - 2 (unsigned ids); vertex ids int32
    assert L.polylla_build_halfedges_ex(fake, V, fake, 1_431_655_765, 0, 0, 0, fake, 0, None, ctypes.byref(h)) == -6
    assert L.polylla_build_halfedges_ex(fake, V, fake, 1_400_000_000, 1000, 0, 0, fake, 0, None, ctypes.byref(h)) == -7
    assert L.polylla_build_halfedges(fake, V, fake, 800_000_000, fake, 0, None, ctypes.byref(h)) == -6  # 6T > 2^32
    assert L.polylla_build_halfedges_ex(fake, 2**31, fake, 10, 0, 0, 0, fake, 0, None, ctypes.byref(h)) == -6
    # a row-stride hint (grid tiling) changes the per-tile arrays only slightly; -1 is invalid
    s = 2000
    Tg = 2 * (s - 1) ** 2
    g = L.polylla_workspace_bytes_ex(s * s, Tg, 4 * (s - 1), 0, 2 * (s - 1))
    assert 0 < g - L.polylla_workspace_bytes_ex(s * s, Tg, 4 * (s - 1), 0, 0) < Tg // 2  # (BB: 3T/8 bytes)
    assert L.polylla_workspace_bytes_ex(s * s, Tg, 4 * (s - 1), 0, -1) == 0


def test_host_only_calls():
    from paper_2403_14723_b200 import polylla as pp
    L = pp.lib()
    assert pp.workspace_bytes(1024, 1922) > 6 * 1922 * 4 * 3
    assert L.polylla_status_string(0) == b"ok"
    assert L.polylla_status_string(-9) == b"frontier loop without a seed"
    # invalid arguments are reported synchronously without touching the GPU
    import ctypes
    h = ctypes.c_void_p()
    assert L.polylla_build_halfedges(None, 0, None, 0, None, 0, None, ctypes.byref(h)) == -1


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2403_14723_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            p = os.path.join(dirpath, f)
            if f.endswith(".py"):
                tree = ast.parse(open(p).read())
                for node in ast.walk(tree):
                    if isinstance(node, (ast.Import, ast.ImportFrom)):
                        names = [a.name for a in node.names] + [getattr(node, "module", None) or ""]
                        assert not any(n.split(".")[0] == "oracle" for n in names), p
            if f.endswith((".cu", ".cuh", ".h")):
                assert "oracle" not in open(p).read().replace("no code", ""), p


def test_oracle_shares_no_code_with_product():
    src = open(os.path.join(ROOT, "oracle", "polylla_oracle.c")).read()
    assert "#include \"" not in src  # only system headers
