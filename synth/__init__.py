"""Seeded synthetic triangulations -- the INPUT GENERATORS shared by both sides.

This module is the one piece of code that both the CPU oracle (``oracle/``) and the
CUDA path (``paper_2403_14723_b200``) consume.  It contains none of the Polylla
method's arithmetic (no lengths, labels, half-edges, walks); it only produces
``(xy, tri)`` inputs shaped like the paper's workloads:

* ``grid(s, a, seed)``      -- Alg. 13 grid; ``a > 0`` jitters
  interior vertices by ``a*(2u-1)`` per axis (BASELINE.json configs 1, 4, 5).
* ``random_delaunay(n, seed, delta)`` -- uniform points in the unit square,
  border snapping within ``delta``, Delaunay-triangulated by an
  exact-predicate incremental builder (replaces the Triangle tool).
* small hand-made fixtures (square of Fig. 5, single triangle, barrier fan,
  tie lattice) used by the unit tests.

Recipes and their citations are in DESIGN.md ("Input recipe").
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynth.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = ctypes.CDLL(path)
        lib.synth_grid.restype = ctypes.c_int64
        lib.synth_grid.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64,
                                   ctypes.c_void_p, ctypes.c_void_p]
        lib.synth_random_delaunay.restype = ctypes.c_int64
        lib.synth_random_delaunay.argtypes = [ctypes.c_int64, ctypes.c_uint64, ctypes.c_double,
                                              ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64]
        lib.synth_rng.restype = ctypes.c_uint64
        lib.synth_rng.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _LIB = lib
    return _LIB


def rng(seed: int, ctr: int) -> int:
    """The shared counter-based generator (splitmix64 finaliser of seed*phi + ctr + 1)."""
    return int(_lib().synth_rng(seed, ctr))


def grid(s: int, a: float = 0.0, seed: int = 0):
    """Alg. 13 grid with s*s vertices and 2(s-1)^2 triangles (all CW in (x, y), R10).

    Vertex k sits at (k div s, k mod s) (+ jitter a*(2u-1) per axis for interior
    vertices when a > 0).  Domain [0, s-1]^2.
    """
    s = int(s)
    n = s * s
    T = 2 * (s - 1) * (s - 1)
    xy = np.empty((n, 2), dtype=np.float64)
    tri = np.empty((T, 3), dtype=np.int32)
    got = _lib().synth_grid(s, float(a), int(seed), xy.ctypes.data, tri.ctypes.data)
    if got != T:
        raise RuntimeError(f"synth_grid failed ({got})")
    return xy, tri


def random_delaunay(n: int, seed: int, delta: float | None = None):
    """Delaunay triangulation of n points in the unit square (ids 0..3 = corners).

    ``delta`` defaults to 1/sqrt(n) (reading R18).  Coordinates are exact
    multiples of 2^-24.  Triangles sorted by Morton code of their centroid, CCW.
    """
    n = int(n)
    if delta is None:
        delta = 1.0 / math.sqrt(n)
    cap = 2 * n + 8
    xy = np.empty((n, 2), dtype=np.float64)
    tri = np.empty((cap, 3), dtype=np.int32)
    T = _lib().synth_random_delaunay(n, int(seed), float(delta), xy.ctypes.data, tri.ctypes.data, cap)
    if T < 0:
        raise RuntimeError(f"synth_random_delaunay failed ({T})")
    return xy, np.ascontiguousarray(tri[:T])


# --------------------------------------------------------------------------- fixtures

def fixture_square():
    """F1: the two-triangle square of PAPER.md Fig. 5 (L274-298)."""
    xy = np.array([[0, 0], [1, 0], [1, 1], [0, 1]], dtype=np.float64)
    tri = np.array([[0, 1, 2], [0, 2, 3]], dtype=np.int32)
    return xy, tri


def fixture_triangle():
    """F2: a single triangle."""
    xy = np.array([[0, 0], [1, 0], [0, 1]], dtype=np.float64)
    tri = np.array([[0, 1, 2]], dtype=np.int32)
    return xy, tri


def fixture_fan():
    """F4: a 5-triangle fan around vertex 0 with one barrier tip (vertex 0, degree 5).

    w_i = r_i (cos t_i, sin t_i), t = 0,72,144,216,288 deg, r = 1.0,1.7,2.9,4.9,2.0;
    triangles (0, i, i%5+1) for i = 1..5 (SURVEY.md 8(c) "F4 barrier fan").
    """
    r = [1.0, 1.7, 2.9, 4.9, 2.0]
    xy = [[0.0, 0.0]]
    for i in range(5):
        t = math.radians(72.0 * i)
        xy.append([r[i] * math.cos(t), r[i] * math.sin(t)])
    tri = [[0, i, i % 5 + 1] for i in range(1, 6)]
    return np.array(xy, dtype=np.float64), np.array(tri, dtype=np.int32)


def fixture_long_fan(n: int, span_deg: float = 300.0):
    """F6: an open fan of n triangles around a hub with slowly growing radii, which is ONE
    polygon of n + 2 vertices (n >= 8: rim chords shorter than spokes): hub h = (0, 0), rim p_i = r_i (cos t_i, sin t_i) with
    r_i = 1 + 1e-4 i and t_i = span * i / n (i = 0..n); triangles (h, p_i, p_{i+1}).  The
    rim chords are short, so the longest edge of triangle i is its spoke h-p_{i+1}, which
    is not the longest edge of triangle i + 1: every interior spoke is non-frontier, the
    Lepp chain runs 0 -> n - 1 and ends at the border spoke h-p_n.  Loops of >= 255
    entries (the emission's escaped length) and > 1024 (the in-tile walk bound)."""
    i = np.arange(n + 1, dtype=np.float64)
    r = 1.0 + 1e-4 * i
    t = np.radians(span_deg) * i / n
    xy = np.concatenate([[[0.0, 0.0]], np.stack([r * np.cos(t), r * np.sin(t)], axis=1)]).astype(np.float64)
    k = np.arange(n, dtype=np.int32)
    tri = np.stack([np.zeros(n, dtype=np.int32), k + 1, k + 2], axis=1).astype(np.int32)
    return np.ascontiguousarray(xy), np.ascontiguousarray(tri)


def fixture_tie_lattice(m: int = 9):
    """F5: lattice with every triangle's longest side tied (sqrt10, sqrt10, 2).

    P(i, j) = (2i + (j mod 2), 3j), i, j < m; even rows (a,b,c),(b,d,c), odd rows
    (a,b,d),(a,d,c) with a=(i,j), b=(i+1,j), c=(i,j+1), d=(i+1,j+1).
    """
    idx = lambda i, j: j * m + i  # noqa: E731
    xy = np.array([[2 * i + (j % 2), 3 * j] for j in range(m) for i in range(m)], dtype=np.float64)
    tri = []
    for j in range(m - 1):
        for i in range(m - 1):
            a, b, c, d = idx(i, j), idx(i + 1, j), idx(i, j + 1), idx(i + 1, j + 1)
            if j % 2 == 0:
                tri += [[a, b, c], [b, d, c]]
            else:
                tri += [[a, b, d], [a, d, c]]
    return xy, np.array(tri, dtype=np.int32)


CONFIGS = {
    # BASELINE.json configs; the recipe for each is stated in DESIGN.md.
    1: dict(kind="jittered", s=32, a=0.2, seed=1),
    2: dict(kind="random", n=1_000_000, seed=2),
    3: dict(kind="random", n=10_000_000, seed=3),
    4: dict(kind="jittered", s=16000, a=0.2, seed=4),
    5: dict(kind="batch", s=2000, a=0.2, count=64),
}


def make(kind: str, **kw):
    if kind == "jittered":
        return grid(kw["s"], kw.get("a", 0.2), kw.get("seed", 0))
    if kind == "regular":
        return grid(kw["s"], 0.0, 0)
    if kind == "random":
        return random_delaunay(kw["n"], kw["seed"], kw.get("delta"))
    raise ValueError(kind)


# --------------------------------------------------------------------------- device generator
_DEV = None


def grid_device(s: int, a: float = 0.0, seed: int = 0, device="cuda", stream=None):
    """Alg. 13 grid generated on the GPU (synth/csrc/gridgen_dev.cu); bit-identical to grid()."""
    import torch

    global _DEV
    if _DEV is None:
        path = os.path.join(_HERE, "libsynth_dev.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        _DEV = ctypes.CDLL(path)
        _DEV.synth_grid_dev.restype = ctypes.c_int
        _DEV.synth_grid_dev.argtypes = [ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_void_p,
                                        ctypes.c_void_p, ctypes.c_void_p]
    s = int(s)
    xy = torch.empty((s * s, 2), dtype=torch.float64, device=device)
    tri = torch.empty((2 * (s - 1) * (s - 1), 3), dtype=torch.int32, device=device)
    st = (stream or torch.cuda.current_stream(xy.device)).cuda_stream
    rc = _DEV.synth_grid_dev(s, float(a), int(seed), xy.data_ptr(), tri.data_ptr(), ctypes.c_void_p(st))
    if rc:
        raise RuntimeError(f"synth_grid_dev failed ({rc})")
    return xy, tri
