"""Pins of the CPU oracle against what the paper and the mathematics fix (not against
itself): hand-worked fixtures, closed forms for Alg. 13 grids, brute-force Lepp
terminal-edge regions (Defs. 1-2), invariants, error kinds.  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
import synth
from checks import canonical, check_output, flip_walk, flood_pieces, lepp_regions

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ----------------------------------------------------------------- F1: the square
def test_square_fig5():
    g = gold("square.json")
    xy = np.array(g["xy"], np.float64)
    tri = np.array(g["tri"], np.int32)
    o = oracle.run(xy, tri)
    assert o["H"] == g["H"] and o["B"] == g["B"]
    assert np.nonzero(o["longest"])[0].tolist() == g["longest"]
    assert np.nonzero(o["frontier0"][:6])[0].tolist() == g["frontier_interior"]
    assert o["seeds0"].tolist() == g["seeds0"]
    assert o["twin"].tolist() == g["twin"]
    assert o["next"].tolist() == g["next"]
    assert o["seeds"].tolist() == g["seeds"]
    assert o["offsets"].tolist() == g["offsets"]
    assert o["loops"].tolist() == g["loops"]
    check_output(xy, tri, o, o["frontier1"])


# ----------------------------------------------------------------- F2: one triangle
def test_single_triangle():
    xy, tri = synth.fixture_triangle()
    o = oracle.run(xy, tri)
    # 3 interior + 3 border half-edges; L157: 1 seed (terminal border edge)
    assert o["H"] == 6 and o["B"] == 3
    assert o["n_seeds0"] == 1 and o["P"] == 1
    assert canonical(o["offsets"], o["loops"]) == [(0, 1, 2)]
    # longest side of (0,0),(1,0),(0,1) is the hypotenuse 1->2 = half-edge 1
    assert np.nonzero(o["longest"])[0].tolist() == [1]
    # border chain is a closed 3-cycle
    nb = o["next"][3:]
    assert sorted(nb.tolist()) == [3, 4, 5]
    check_output(xy, tri, o, o["frontier1"])


def test_cw_input_is_reoriented():
    """CW triangles are silently re-oriented (swap v1, v2)."""
    xy, tri = synth.fixture_square()
    o1 = oracle.run(xy, tri)
    o2 = oracle.run(xy, tri[:, [0, 2, 1]])
    assert o2["flips"] == 2 and o1["flips"] == 0
    assert np.array_equal(o1["origin"], o2["origin"])
    assert canonical(o1["offsets"], o1["loops"]) == canonical(o2["offsets"], o2["loops"])


# ----------------------------------------------------------------- F3: grids
def test_grid3_alg13():
    g = gold("grid3.json")
    xy, tri = synth.grid(3)
    assert tri.shape[0] == g["n_triangles"]
    o = oracle.run(xy, tri)
    assert o["H"] == g["H"] and o["B"] == g["B"]
    assert canonical(o["offsets"], o["loops"]) == [tuple(x) for x in g["canonical_loops"]]


@pytest.mark.parametrize("s", [2, 3, 10, 32, 50, 101])
def test_grid_closed_forms(s):
    """Alg. 13 grids: every cell diagonal is strictly longest in
    both triangles, so each cell is one region: P = (s-1)^2 quads, F0 interior =
    4(s-1)^2 half-edges (2 legs per triangle), seeds = (s-1)^2, B = 4(s-1), no tips
    (Table 2-3 'Rep' = 0.0)."""
    xy, tri = synth.grid(s)
    o = oracle.run(xy, tri)
    c = (s - 1) ** 2
    assert o["flips"] == 2 * c  # all Alg. 13 triangles are CW (R10)
    assert o["B"] == 4 * (s - 1) and o["H"] == 3 * 2 * c + 4 * (s - 1)
    assert int(o["frontier0"][:6 * c].sum()) == 4 * c
    assert o["n_seeds0"] == c and o["P"] == c and o["n_tips"] == 0
    assert o["L"] == 4 * c
    assert np.all(np.diff(o["offsets"]) == 4)
    # each polygon is a unit cell
    for lp in canonical(o["offsets"], o["loops"]):
        v = lp[0]
        assert lp == (v, v + s, v + s + 1, v + 1)
    # Euler for a disk: V - E + F = 1
    assert xy.shape[0] - o["H"] // 2 + tri.shape[0] == 1


def test_grid_2000_counts():
    """Config-5 regular grid closed form: P = 1999^2 = 3,996,001, L = 4 P."""
    xy, tri = synth.grid(2000)
    o = oracle.run(xy, tri)
    assert o["P"] == 3_996_001 and o["L"] == 15_984_004 and o["n_tips"] == 0


# ----------------------------------------------------------------- F4: barrier fan
def test_fan_barrier_tip_repair():
    g = gold("fan.json")
    xy, tri = synth.fixture_fan()
    o = oracle.run(xy, tri)
    assert np.nonzero(o["longest"])[0].tolist() == g["longest"]
    assert o["tips"].tolist() == g["tips"]
    assert canonical(o["offsets"], o["loops"]) == [tuple(x) for x in g["canonical_loops"]]
    # pre-repair: one region, one seed, a single loop with the barrier 1->0->1
    assert o["n_seeds0"] == 1
    check_output(xy, tri, o, o["frontier1"])


# ----------------------------------------------------------------- F6: long open fan
@pytest.mark.parametrize("n", [12, 40, 300])
def test_long_fan_closed_form(n):
    """synth.fixture_long_fan: the longest edge of triangle i is its spoke h-p_{i+1} (the
    rim chords are shorter, r grows with i), so Lcode = 2 for every triangle (half-edge
    3i + 2 runs p_{i+1} -> h), every interior spoke is non-frontier and the whole fan is
    one terminal region whose terminal edge is the border spoke h-p_n (Def. 2): one polygon,
    the loop h, p_0, ..., p_n (vertex ids 0..n+1), no barrier tip."""
    xy, tri = synth.fixture_long_fan(n)
    o = oracle.run(xy, tri)
    assert o["lcode"].tolist() == [2] * n
    assert o["P"] == 1 and o["n_tips"] == 0 and o["B"] == n + 2
    assert o["loops"].tolist() == list(range(n + 2))
    check_output(xy, tri, o, o["frontier1"])


# ----------------------------------------------------------------- F5: tie lattice
def test_tie_lattice_matches_bruteforce_lepp():
    """Every triangle has two tied longest sides; the tie-break (first max, R7)
    decides the regions.  The brute-force Lepp count pins the polygon count."""
    xy, tri = synth.fixture_tie_lattice()
    regions, _ = lepp_regions(xy, tri)
    o = oracle.run(xy, tri)
    assert o["n_tips"] == 0
    assert o["P"] == len(regions) == 8
    check_output(xy, tri, o, o["frontier1"])


# ----------------------------------------------------------------- brute-force Lepp
def _corpus():
    rng = np.random.default_rng(123)
    out = []
    for i, n in enumerate([8, 12, 20, 30, 50, 80, 120, 200, 350, 600]):
        xy, tri = synth.random_delaunay(n, 1000 + i)
        out.append((f"del{n}", xy, tri))
        out.append((f"flip{n}", xy, flip_walk(xy, tri, max(3, tri.shape[0] // 3), rng)))
    for s in (4, 7, 12):
        xy, tri = synth.grid(s, 0.2, s)
        out.append((f"jit{s}", xy, tri))
    return out


@pytest.mark.parametrize("name,xy,tri", _corpus(), ids=lambda v: v if isinstance(v, str) else "")
def test_prerepair_partition_equals_lepp_regions(name, xy, tri):
    """Defs. 1-2: the partition of triangles
    obtained by flooding across non-frontier edges (F0) equals the terminal-edge
    regions enumerated by brute force; #seeds = #regions = #pre-repair loops."""
    regions, _ = lepp_regions(xy, tri)
    o = oracle.run(xy, tri)
    T = tri.shape[0]
    pieces = flood_pieces(T, o["twin"], o["frontier0"])
    assert set(pieces) == set(regions)
    assert o["n_seeds0"] == len(regions)
    # each pre-repair loop bounds exactly one region: its half-edges' triangles
    # lie in one region, and every interior F0 half-edge is on one loop
    nxt = o["next_pre"]
    region_of = {t: i for i, g in enumerate(regions) for t in g}
    seen = np.zeros(o["H"], bool)
    for s in o["seeds0"].tolist():
        # rotate the seed about its origin (sweep_out on the input mesh) to a frontier
        x = s
        while not o["frontier0"][x]:
            x = (3 * (o["twin"][x] // 3)) + ((o["twin"][x] % 3) + 1) % 3
        r = region_of[x // 3]
        y = x
        while True:
            assert region_of[y // 3] == r
            assert not seen[y]
            seen[y] = True
            y = nxt[y]
            if y == x:
                break
    assert np.array_equal(seen[:3 * T], o["frontier0"][:3 * T].astype(bool))
    info = check_output(xy, tri, o, o["frontier1"])
    assert info["repeated_vertex_loops"] >= 0


@pytest.mark.parametrize("name,xy,tri", _corpus()[::3], ids=lambda v: v if isinstance(v, str) else "")
def test_triangle_regions_label_the_lepp_partition(name, xy, tri):
    """oracle.triangle_regions (NEXT-4, pre-repair): its label classes are exactly the
    brute-force terminal-edge regions of Defs. 1-2 and each label is the smallest
    triangle id of its region."""
    regions, _ = lepp_regions(xy, tri)
    lab = oracle.triangle_regions(oracle.run(xy, tri))
    assert len(set(lab.tolist())) == len(regions)
    for g in regions:
        ids = sorted(g)
        assert set(lab[ids].tolist()) == {ids[0]}


def test_triangle_regions_closed_forms():
    """Alg. 13 grids: every cell (triangles 2c, 2c+1, sharing their hypotenuse) is one
    terminal-edge region -> label t - t % 2; the square is one region; the barrier fan is
    one region before the repair (its two polygons come from the repair)."""
    for s in (2, 3, 9):
        lab = oracle.triangle_regions(oracle.run(*synth.grid(s)))
        t = np.arange(2 * (s - 1) ** 2)
        assert np.array_equal(lab, t - t % 2)
    assert oracle.triangle_regions(oracle.run(*synth.fixture_square())).tolist() == [0, 0]
    assert oracle.triangle_regions(oracle.run(*synth.fixture_fan())).tolist() == [0] * 5


def test_repair_splits_are_region_subsets():
    """Repair (Alg. 6) only splits regions: each final polygon's flood piece (F1)
    lies inside one Lepp region, and every region is the union of its pieces."""
    xy, tri = synth.random_delaunay(3000, 77)
    regions, _ = lepp_regions(xy, tri)
    o = oracle.run(xy, tri)
    assert o["n_tips"] > 0
    pieces = flood_pieces(tri.shape[0], o["twin"], o["frontier1"])
    region_of = {t: i for i, g in enumerate(regions) for t in g}
    for g in pieces:
        assert len({region_of[t] for t in g}) == 1
    assert len(pieces) == o["P"]
    check_output(xy, tri, o, o["frontier1"])


def test_tips_have_one_frontier_edge_and_middle_edges_are_new():
    """Barrier tips: exactly one incident F0 edge; after repair no
    vertex has exactly one incident frontier edge (F1)."""
    xy, tri = synth.random_delaunay(5000, 9)
    o = oracle.run(xy, tri)
    origin, f0, f1 = o["origin"], o["frontier0"], o["frontier1"]
    V = xy.shape[0]
    cnt0 = np.bincount(origin[f0.astype(bool)], minlength=V)
    cnt1 = np.bincount(origin[f1.astype(bool)], minlength=V)
    # outgoing frontier half-edges count the incident frontier edges of interior vertices
    assert sorted(o["tips"].tolist()) == sorted(np.nonzero(cnt0 == 1)[0].tolist())
    assert np.count_nonzero(cnt1 == 1) == 0
    assert o["n_mid"] == o["n_tips"]
    assert int(f1.sum() - f0.sum()) <= 2 * o["n_mid"]


def test_determinism():
    xy, tri = synth.random_delaunay(20000, 5)
    a = oracle.run(xy, tri)
    b = oracle.run(xy, tri)
    for k in ("origin", "twin", "next", "prev", "seeds", "offsets", "loops"):
        assert np.array_equal(a[k], b[k])


def test_prev_is_inverse_on_frontier_and_border():
    xy, tri = synth.random_delaunay(2000, 6)
    o = oracle.run(xy, tri)
    T = tri.shape[0]
    f1 = o["frontier1"].astype(bool)
    e = np.nonzero(f1)[0]
    assert np.array_equal(o["prev"][o["next"][e]], e)
    nf = np.nonzero(~f1[:3 * T])[0]
    assert np.array_equal(o["prev"][nf], 3 * (nf // 3) + (nf % 3 + 2) % 3)


# ----------------------------------------------------------------- error kinds
def _err(xy, tri):
    with pytest.raises(oracle.OracleError) as ei:
        oracle.run(np.asarray(xy, np.float64), np.asarray(tri, np.int32))
    return oracle.STATUS[ei.value.code]


def test_errors():
    sq_xy, _ = synth.fixture_square()
    assert _err(sq_xy, [[0, 1, 7]]) == "DANGLING_INDEX"
    assert _err([[0, 0], [1, 0], [2, 0]], [[0, 1, 2]]) == "DEGENERATE_TRI"
    assert _err(sq_xy, [[0, 1, 1]]) == "DEGENERATE_TRI"
    # an edge 0-1 in three triangles
    assert _err([[0, 0], [1, 0], [0.5, 1], [0.5, -1], [0.5, 2]],
                [[0, 1, 2], [1, 0, 3], [0, 1, 4]]) == "NON_MANIFOLD_EDGE"
    # the same directed edge twice (overlapping triangles)
    assert _err([[0, 0], [1, 0], [0.5, 1], [0.5, 2]], [[0, 1, 2], [0, 1, 3]]) == "NON_MANIFOLD_EDGE"
    # bow-tie: two triangles sharing only vertex 0
    assert _err([[0, 0], [1, 0], [1, 1], [-1, 0], [-1, -1]], [[0, 1, 2], [0, 3, 4]]) == "NON_MANIFOLD_VERTEX"


# ---- per-triangle polygon ids (oracle.triangle_polygons)

def _signed_area2(xy, a, b, c):
    return (xy[b, 0] - xy[a, 0]) * (xy[c, 1] - xy[a, 1]) - (xy[b, 1] - xy[a, 1]) * (xy[c, 0] - xy[a, 0])


@pytest.mark.parametrize("s", [2, 3, 10])
def test_triangle_polygons_grid_closed_form(s):
    # Alg. 13 emits the two triangles of each cell together; every cell is one quad
    # (closed form of test_grid_closed_forms), so triangle t lies in polygon t // 2
    xy, tri = synth.grid(s)
    o = oracle.triangle_polygons(oracle.run(xy, tri))
    np.testing.assert_array_equal(o, np.arange(tri.shape[0]) // 2)


def test_triangle_polygons_fixtures():
    # square (Fig. 5): one polygon; fan F4: loops (0,1,2,3,4) <- triangles
    # (0,1,2),(0,2,3),(0,3,4) and (0,4,5,1) <- (0,4,5),(0,5,1)
    np.testing.assert_array_equal(oracle.triangle_polygons(oracle.run(*synth.fixture_square())), [0, 0])
    np.testing.assert_array_equal(oracle.triangle_polygons(oracle.run(*synth.fixture_fan())), [0, 0, 0, 1, 1])
    np.testing.assert_array_equal(oracle.triangle_polygons(oracle.run(*synth.fixture_triangle())), [0])


@pytest.mark.parametrize("kind,arg,seed", [("random", 3000, 4), ("jittered", 40, 2)])
def test_triangle_polygons_areas(kind, arg, seed):
    # every polygon's loop area (shoelace) = the summed area of the triangles assigned to it,
    # and every polygon owns at least one triangle (no holes: one loop per piece)
    xy, tri = synth.random_delaunay(arg, seed) if kind == "random" else synth.grid(arg, 0.2, seed)
    r = oracle.run(xy, tri)
    o = oracle.triangle_polygons(r)
    P = r["P"]
    assert o.min() == 0 and o.max() == P - 1 and len(np.unique(o)) == P
    t = r["origin"][:3 * r["T"]].reshape(-1, 3)
    ta = _signed_area2(xy, t[:, 0], t[:, 1], t[:, 2])
    assert (ta > 0).all()
    tri_sum = np.bincount(o, weights=ta, minlength=P)
    off, lp = r["offsets"], r["loops"]
    nxt_idx = np.arange(len(lp)) + 1
    poly_of_entry = np.repeat(np.arange(P), np.diff(off))
    nxt_idx[off[1:] - 1] = off[:-1]  # wrap each loop
    a, b = lp, lp[nxt_idx]
    shoe = np.bincount(poly_of_entry, weights=xy[a, 0] * xy[b, 1] - xy[b, 0] * xy[a, 1], minlength=P)
    np.testing.assert_allclose(shoe, tri_sum, rtol=1e-9, atol=1e-12 * np.abs(ta).max())
