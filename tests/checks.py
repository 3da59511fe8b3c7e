"""Independent checkers used by the tests (test infrastructure; no product code).

* ``lepp_regions``     -- brute-force Longest-Edge Propagation Path regions straight
  from Defs. 1-2, on a triangle-adjacency dict built here.
* ``flood_pieces``     -- triangles grouped by flooding across non-frontier edges.
* ``canonical``        -- canonical polygon list (north_star): each loop rotated to its
  minimum vertex (ties: smallest successor), polygons sorted.
* ``check_output``     -- the invariants of SPEC.md L187-193 / north_star on any output.
"""
from __future__ import annotations

import numpy as np


def orient_tris(xy, tri):
    """CCW orientation by the signed-area rule (swap v1, v2 when negative; R10)."""
    out = []
    for a, b, c in tri.tolist():
        ar = (xy[b, 0] - xy[a, 0]) * (xy[c, 1] - xy[a, 1]) - (xy[b, 1] - xy[a, 1]) * (xy[c, 0] - xy[a, 0])
        out.append((a, c, b) if ar < 0 else (a, b, c))
    return out


def lepp_regions(xy, tri):
    """Terminal-edge regions by brute force (Def. 1: follow the neighbour across the
    longest edge until the longest edge is shared-longest or on the border; Def. 2:
    group triangles by terminal edge).  Longest edge = first maximum of the squared
    lengths of (v0v1, v1v2, v2v0) after orientation (R7).  Returns a list of frozensets
    of triangle ids and the list of terminal edges (as frozensets of 2 vertices)."""
    tris = orient_tris(xy, tri)
    adj = {}
    for t, (a, b, c) in enumerate(tris):
        for u, v in ((a, b), (b, c), (c, a)):
            adj.setdefault(frozenset((u, v)), []).append(t)

    def longest(t):
        a, b, c = tris[t]
        best, bl = None, -1.0
        for u, v in ((a, b), (b, c), (c, a)):
            dx = xy[v, 0] - xy[u, 0]
            dy = xy[v, 1] - xy[u, 1]
            d = dx * dx + dy * dy
            if d > bl:
                best, bl = frozenset((u, v)), d
        return best

    L = [longest(t) for t in range(len(tris))]
    term = []
    for t0 in range(len(tris)):
        t, seen = t0, set()
        while True:
            if t in seen:
                raise RuntimeError("Lepp cycle (exact tie loop, reading R12)")
            seen.add(t)
            e = L[t]
            nbrs = [u for u in adj[e] if u != t]
            if not nbrs:
                term.append(e)  # terminal border edge
                break
            u = nbrs[0]
            if L[u] == e:
                term.append(e)  # terminal edge shared-longest by t and u
                break
            t = u
    groups = {}
    for t, e in enumerate(term):
        groups.setdefault(e, set()).add(t)
    return [frozenset(g) for g in groups.values()], list(groups.keys())


def flood_pieces(T, twin, frontier):
    """Union triangles across interior half-edges that are not frontier."""
    parent = list(range(T))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    tw = np.asarray(twin)
    fr = np.asarray(frontier)
    for e in range(3 * T):
        if not fr[e] and tw[e] < 3 * T:
            a, b = find(e // 3), find(int(tw[e]) // 3)
            if a != b:
                parent[a] = b
    groups = {}
    for t in range(T):
        groups.setdefault(find(t), set()).add(t)
    return [frozenset(g) for g in groups.values()]


def loops_of(offsets, loops):
    o = np.asarray(offsets)
    lp = np.asarray(loops)
    return [lp[o[i]:o[i + 1]].tolist() for i in range(len(o) - 1)]


def canonical(offsets, loops):
    """Rotate each loop to start at its minimum vertex (if it repeats, the occurrence
    with the smallest successor) and sort the polygons (north_star canonical form)."""
    out = []
    for lp in loops_of(offsets, loops):
        n = len(lp)
        m = min(lp)
        best = None
        for i, v in enumerate(lp):
            if v == m:
                cand = lp[i:] + lp[:i]
                if best is None or cand[1 % n] < best[1 % n]:
                    best = cand
        out.append(tuple(best))
    out.sort()
    return out


def poly_area(xy, lp):
    x = xy[lp, 0]
    y = xy[lp, 1]
    return 0.5 * float(np.sum(x * np.roll(y, -1) - np.roll(x, -1) * y))


def tri_area(xy, tris, t):
    a, b, c = tris[t]
    return 0.5 * ((xy[b, 0] - xy[a, 0]) * (xy[c, 1] - xy[a, 1]) - (xy[b, 1] - xy[a, 1]) * (xy[c, 0] - xy[a, 0]))


def check_output(xy, tri, out, frontier1=None, area_check=True):
    """Invariants (north_star):
    mesh-core (twin involution, origin(next e) = target e), no barrier tip
    (next(e) != twin(e) on loops), every interior frontier half-edge on exactly one
    loop, seeds strictly increasing and minimal on their loops, loops start at
    origin[seed], area conservation (and per-polygon area = its flood piece's area
    when frontier1 is given).  Returns a dict of counts (repeated-vertex loops)."""
    T = tri.shape[0]
    origin = np.asarray(out["origin"]); twin = np.asarray(out["twin"]); nxt = np.asarray(out["next"])
    H = origin.shape[0]
    seeds = np.asarray(out["seeds"]); offsets = np.asarray(out["offsets"]); loops = np.asarray(out["loops"])
    ids = np.arange(H)
    assert np.all(twin[twin] == ids), "twin not an involution"
    assert np.all(twin != ids)
    assert np.all(origin[nxt] == origin[twin]), "origin(next e) != target(e)"
    assert np.all(np.diff(seeds) > 0), "seeds not strictly increasing"
    on_loop = np.zeros(H, np.int64)
    repeated = 0
    P = seeds.shape[0]
    assert offsets.shape[0] == P + 1 and offsets[0] == 0 and offsets[-1] == loops.shape[0]
    for p in range(P):
        s = int(seeds[p])
        x, k, mn = s, 0, s
        verts = []
        while True:
            assert x < 3 * T, "loop leaves the interior"
            assert nxt[x] != twin[x], "barrier tip survived (next == twin)"
            on_loop[x] += 1
            verts.append(int(origin[x]))
            mn = min(mn, x)
            x = int(nxt[x]); k += 1
            if x == s:
                break
            assert k <= H
        assert mn == s, "seed is not the minimum half-edge of its loop"
        assert verts == loops[offsets[p]:offsets[p + 1]].tolist()
        if len(set(verts)) != len(verts):
            repeated += 1
    assert on_loop.max(initial=0) <= 1, "half-edge on two loops"
    if frontier1 is not None:
        f1 = np.asarray(frontier1)[:3 * T].astype(bool)
        assert np.array_equal(on_loop[:3 * T] == 1, f1), "interior frontier half-edges != loop half-edges"
    # every border edge appears on exactly one loop (through its interior half)
    inner_of_border = twin[3 * T:]
    assert np.all(on_loop[inner_of_border] == 1)
    if area_check:
        tris = orient_tris(xy, tri)
        tot = sum(tri_area(xy, tris, t) for t in range(T))
        pa = sum(poly_area(xy, lp) for lp in loops_of(offsets, loops))
        assert abs(pa - tot) <= 1e-9 * abs(tot), (pa, tot)
        if frontier1 is not None:
            pieces = flood_pieces(T, twin, frontier1)
            piece_of = {}
            for i, g in enumerate(pieces):
                for t in g:
                    piece_of[t] = i
            assert len(pieces) == P, (len(pieces), P)
            for p in range(P):
                s = int(seeds[p])
                g = pieces[piece_of[s // 3]]
                a_piece = sum(tri_area(xy, tris, t) for t in g)
                a_poly = poly_area(xy, loops[offsets[p]:offsets[p + 1]])
                assert abs(a_piece - a_poly) <= 1e-9 * max(abs(a_piece), 1e-300), (p, a_piece, a_poly)
    return dict(repeated_vertex_loops=repeated)


def flip_walk(xy, tri, n_flips, rng):
    """Random legal edge flips of a CCW triangulation (non-Delaunay inputs, PAPER.md L45
    'any triangulation').  A flip of the edge a-b shared by (a,b,c) and (b,a,d) into
    (a,d,c),(d,b,c) is applied only when both new triangles have positive area."""
    tris = [list(t) for t in orient_tris(xy, tri)]

    def area(a, b, c):
        return (xy[b, 0] - xy[a, 0]) * (xy[c, 1] - xy[a, 1]) - (xy[b, 1] - xy[a, 1]) * (xy[c, 0] - xy[a, 0])

    done = 0
    for _ in range(20 * n_flips):
        if done >= n_flips:
            break
        edges = {}
        for t, (a, b, c) in enumerate(tris):
            for k, (u, v) in enumerate(((a, b), (b, c), (c, a))):
                edges[(u, v)] = (t, k)
        t1 = int(rng.integers(len(tris)))
        k1 = int(rng.integers(3))
        a, b = tris[t1][k1], tris[t1][(k1 + 1) % 3]
        c = tris[t1][(k1 + 2) % 3]
        if (b, a) not in edges:
            continue
        t2, k2 = edges[(b, a)]
        d = tris[t2][(k2 + 2) % 3]
        if area(a, d, c) > 0 and area(d, b, c) > 0:
            tris[t1] = [a, d, c]
            tris[t2] = [d, b, c]
            done += 1
    return np.array(tris, dtype=np.int32)
