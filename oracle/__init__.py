"""ctypes shim over ``oracle/liboracle.so`` -- the sequential CPU Polylla oracle.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this package.
The product package ``paper_2403_14723_b200`` never imports it, and the oracle shares
no code with the CUDA path (see the header of ``polylla_oracle.c``).

Parity pins (what the oracle is checked against, independently of itself) live in
``tests/test_oracle_pins.py``: hand-worked fixtures (Fig. 5, SPEC.md
examples), closed forms for Alg. 13 grids, brute-force Lepp terminal-edge regions
(Defs. 1-2), and invariants.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS = {
    0: "OK", -1: "INVALID_ARGUMENT", -2: "DANGLING_INDEX", -3: "DEGENERATE_TRI",
    -4: "NON_MANIFOLD_EDGE", -5: "NON_MANIFOLD_VERTEX", -6: "INDEX_OVERFLOW",
    -8: "WALK_BOUND", -9: "UNSEEDED_LOOP", -12: "NOMEM",
}

PHASES = ("Build", "LM", "LF", "LS", "Trav", "Rep", "Extract", "Total")


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code} ({STATUS.get(code, '?')})")
        self.code = code


class _IO(ctypes.Structure):
    _fields_ = [
        ("T", ctypes.c_int64), ("V", ctypes.c_int64),
        ("xy", ctypes.c_void_p), ("tri", ctypes.c_void_p),
        ("origin", ctypes.c_void_p), ("twin", ctypes.c_void_p),
        ("next", ctypes.c_void_p), ("prev", ctypes.c_void_p),
        ("next_pre", ctypes.c_void_p),
        ("lcode", ctypes.c_void_p), ("longest", ctypes.c_void_p),
        ("frontier0", ctypes.c_void_p), ("frontier1", ctypes.c_void_p),
        ("seeds0", ctypes.c_void_p), ("seeds", ctypes.c_void_p),
        ("offsets", ctypes.c_void_p), ("loops", ctypes.c_void_p),
        ("tips", ctypes.c_void_p),
        ("counts", ctypes.c_int64 * 10), ("times", ctypes.c_double * 8),
        ("hcap", ctypes.c_int64),
    ]


_PATH = os.path.join(_HERE, "liboracle.so")


def use_native() -> str:
    """Switch to a copy of the oracle compiled on THIS host with -O3 -march=native
    -ffp-contract=off (the timing build of SURVEY.md 8(d); no FMA, so bit-identical
    results), cached in a temporary directory.  Returns its path."""
    global _LIB, _PATH
    import subprocess
    import tempfile
    src = os.path.join(_HERE, "polylla_oracle.c")
    out = os.path.join(tempfile.gettempdir(), f"liboracle_native_{os.getuid()}_{int(os.path.getmtime(src))}.so")
    if not os.path.exists(out):
        subprocess.run(["gcc", "-O3", "-march=native", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                        "-o", out + ".tmp", src], check=True)
        os.replace(out + ".tmp", out)
    _PATH, _LIB = out, None
    return out


def _lib():
    global _LIB
    if _LIB is None:
        path = _PATH
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(path)
        lib.oracle_run.restype = ctypes.c_int
        lib.oracle_run.argtypes = [ctypes.POINTER(_IO)]
        lib.oracle_build.restype = ctypes.c_int
        lib.oracle_build.argtypes = [ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                     ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                     ctypes.c_void_p]
        _LIB = lib
    return _LIB


def build(xy: np.ndarray, tri: np.ndarray):
    """Half-edge build only: returns dict origin/twin/next/prev, H, B, flips."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    V, T = xy.shape[0], tri.shape[0]
    cap = max(6 * T, 1)
    origin = np.empty(cap, np.int32); twin = np.empty(cap, np.int32)
    nxt = np.empty(cap, np.int32); prv = np.empty(cap, np.int32)
    hb = np.zeros(3, np.int64)
    rc = _lib().oracle_build(V, xy.ctypes.data, T, tri.ctypes.data, origin.ctypes.data, twin.ctypes.data,
                             nxt.ctypes.data, prv.ctypes.data, hb.ctypes.data)
    if rc:
        raise OracleError(rc)
    H = int(hb[0])
    return dict(origin=origin[:H], twin=twin[:H], next=nxt[:H], prev=prv[:H], H=H, B=int(hb[1]),
                flips=int(hb[2]))


def run(xy: np.ndarray, tri: np.ndarray, hcap: int | None = None):
    """Full sequential Polylla (Alg. 1).  Returns a dict of numpy arrays + counts + times.
    hcap: capacity of the [H] arrays when the caller knows a bound on H = 3T + B (the
    default 6T covers any mesh; huge meshes pass a tight bound to fit host memory)."""
    xy = np.ascontiguousarray(xy, dtype=np.float64)
    tri = np.ascontiguousarray(tri, dtype=np.int32)
    V, T = xy.shape[0], tri.shape[0]
    H = int(hcap) if hcap else 6 * max(T, 1)
    a = dict(
        origin=np.empty(H, np.int32), twin=np.empty(H, np.int32), next=np.empty(H, np.int32),
        prev=np.empty(H, np.int32), next_pre=np.empty(H, np.int32),
        lcode=np.empty(max(T, 1), np.uint8), longest=np.empty(H, np.uint8),
        frontier0=np.empty(H, np.uint8), frontier1=np.empty(H, np.uint8),
        seeds0=np.empty(H, np.int32), seeds=np.empty(max(T, 1), np.int32),
        offsets=np.empty(max(T, 1) + 1, np.int32), loops=np.empty(3 * max(T, 1), np.int32),
        tips=np.empty(max(V, 1), np.int32),
    )
    io = _IO()
    io.T, io.V = T, V
    io.hcap = H
    io.xy, io.tri = xy.ctypes.data, tri.ctypes.data
    for k, v in a.items():
        setattr(io, k, v.ctypes.data)
    rc = _lib().oracle_run(ctypes.byref(io))
    if rc:
        raise OracleError(rc)
    c = list(io.counts)
    H, B, flips, n_seeds0, P, L, n_tips, n_mid = c[:8]
    out = dict(
        H=H, B=B, T=T, V=V, flips=flips, P=P, L=L, n_tips=n_tips, n_mid=n_mid, n_seeds0=n_seeds0,
        origin=a["origin"][:H], twin=a["twin"][:H], next=a["next"][:H], prev=a["prev"][:H],
        next_pre=a["next_pre"][:H], lcode=a["lcode"][:T], longest=a["longest"][:H],
        frontier0=a["frontier0"][:H], frontier1=a["frontier1"][:H], seeds0=a["seeds0"][:n_seeds0],
        seeds=a["seeds"][:P], offsets=a["offsets"][:P + 1], loops=a["loops"][:L], tips=a["tips"][:n_tips],
        times=dict(zip(PHASES, list(io.times))),
    )
    return out


def triangle_polygons(ref: dict):
    """Per-triangle polygon id, from a ``run`` result, by the
    definition: the output polygons are unions of triangles (the terminal-edge regions of
    PAPER.md L76-L128, split by the repair's middle edges).  A piece is a
    connected component of the triangles joined across interior non-frontier (F1 = 0)
    edges (library routine: scipy's connected_components); polygon p bounds the pieces of
    the triangles of its loop's half-edges (walked from seeds[p] along next);
    poly_of_tri[t] = the smallest p bounding t's piece (several loops bound one piece only
    around a hole).  Python loop over the loop entries: small and medium meshes only."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components

    T = ref["T"]
    e = np.arange(3 * T)
    tw = ref["twin"][:3 * T].astype(np.int64)
    m = (ref["frontier1"][:3 * T] == 0) & (tw < 3 * T) & (e < tw)
    g = sp.coo_matrix((np.ones(int(m.sum())), (e[m] // 3, tw[m] // 3)), shape=(T, T))
    _, comp = connected_components(g, directed=False)
    best = np.full(comp.max() + 1, -1, np.int64)
    nxt = ref["next"]
    for p, s in enumerate(ref["seeds"].tolist()):
        x = s
        while True:
            c = comp[x // 3]
            if best[c] < 0:  # p ascends: the first polygon to reach a piece is its smallest
                best[c] = p
            x = int(nxt[x])
            if x == s:
                break
    return best[comp].astype(np.int32)


def triangle_regions(ref: dict):
    """Per-triangle terminal-edge-region label (pre-repair), from a
    ``run`` result, by the definition: the terminal-edge regions of PAPER.md Defs. 1-2
    (L121-128) are the connected components of the triangles joined across interior
    non-frontier edges of the label-phase frontier F0 (pinned against a brute-force
    enumeration of Defs. 1-2 in tests/test_oracle_pins.py); label = the smallest triangle
    id of the component (library routine: scipy's connected_components)."""
    import scipy.sparse as sp
    from scipy.sparse.csgraph import connected_components

    T = ref["T"]
    e = np.arange(3 * T)
    tw = ref["twin"][:3 * T].astype(np.int64)
    m = (ref["frontier0"][:3 * T] == 0) & (tw < 3 * T) & (e < tw)
    g = sp.coo_matrix((np.ones(int(m.sum())), (e[m] // 3, tw[m] // 3)), shape=(T, T))
    _, comp = connected_components(g, directed=False)
    first = np.full(comp.max() + 1, T, np.int64)
    np.minimum.at(first, comp, np.arange(T))
    return first[comp].astype(np.int32)
