"""Parity of the CUDA path (through the C ABI) with the CPU oracle, element by element.

Integer/index outputs must be bit-exact: origin, twin, next (pre- and post-repair),
Lcode, frontier/seed bit-vectors, barrier tips, canonical seeds, CSR offsets and
loops.  The FP64 decisions (orientation sign, longest edge) are taken in the same
precision with the same formula and no FMA on both sides (R11), so they agree exactly.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from checks import canonical, check_output, flip_walk

pytestmark = pytest.mark.gpu


def _pp():
    from paper_2403_14723_b200 import polylla
    return polylla


def bits_to_bool(words, n):
    w = np.ascontiguousarray(words.cpu().numpy()).view(np.uint8)
    return np.unpackbits(w, bitorder="little")[:n].astype(bool)


def gpu_run(xy, tri, **kw):
    pp = _pp()
    return pp.run(torch.from_numpy(np.ascontiguousarray(xy)).cuda(),
                  torch.from_numpy(np.ascontiguousarray(tri, dtype=np.int32)).cuda(), **kw)


def assert_parity(xy, tri, stages=True, invariants=True):
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, debug=stages, prev=True)
    T = tri.shape[0]
    assert res["H"] == ref["H"] and res["n_border"] == ref["B"]
    assert res["n_flips"] == ref["flips"]
    for k in ("origin", "twin", "next", "prev"):
        np.testing.assert_array_equal(res[k].cpu().numpy(), ref[k], err_msg=k)
    np.testing.assert_array_equal(res["seeds"].cpu().numpy(), ref["seeds"])
    np.testing.assert_array_equal(res["offsets"].cpu().numpy(), ref["offsets"])
    np.testing.assert_array_equal(res["loops"].cpu().numpy(), ref["loops"])
    assert res["n_tips"] == ref["n_tips"]
    if stages:
        np.testing.assert_array_equal(res["lcode"].cpu().numpy(), ref["lcode"])
        np.testing.assert_array_equal(bits_to_bool(res["frontier0"], 3 * T), ref["frontier0"][:3 * T].astype(bool))
        np.testing.assert_array_equal(bits_to_bool(res["frontier1"], 3 * T), ref["frontier1"][:3 * T].astype(bool))
        sb = np.nonzero(bits_to_bool(res["seed_bits"], 3 * T))[0]
        np.testing.assert_array_equal(sb, ref["seeds0"])
        np.testing.assert_array_equal(res["next_pre"].cpu().numpy(), ref["next_pre"])
        # tips: GPU records the incoming frontier half-edge e of each tip v = target(e)
        tw = ref["twin"]
        tips_v = np.sort(ref["origin"][tw[res["tips"].cpu().numpy()]])
        np.testing.assert_array_equal(tips_v, np.sort(ref["tips"]))
    assert canonical(res["offsets"].cpu().numpy(), res["loops"].cpu().numpy()) == canonical(ref["offsets"], ref["loops"])
    if invariants:
        out = {k: res[k].cpu().numpy() for k in ("origin", "twin", "next", "seeds", "offsets", "loops")}
        check_output(xy, tri, out, ref["frontier1"], area_check=T <= 50000)
    return res, ref


def test_square():
    assert_parity(*synth.fixture_square())


def test_single_triangle():
    assert_parity(*synth.fixture_triangle())


def test_fan_repair():
    res, ref = assert_parity(*synth.fixture_fan())
    assert res["n_tips"] == 1 and res["P"] == 2


def test_tie_lattice():
    res, _ = assert_parity(*synth.fixture_tie_lattice())
    assert res["P"] == 8


@pytest.mark.parametrize("n", [252, 253, 300, 1100, 2040])
def test_long_fan_one_polygon(n):
    """One polygon of n + 2 vertices (synth.fixture_long_fan): loop lengths around the
    byte code's escape (>= 255: counted by walking at emission) and past the in-tile walk
    bound (> 1024: the global seed walk), alone and next to a random mesh in other tiles."""
    xy, tri = synth.fixture_long_fan(n)
    res, _ = assert_parity(xy, tri)
    assert res["P"] == 1 and int(res["offsets"][1]) == n + 2
    xr, tr = synth.random_delaunay(20000, 11)
    xy2 = np.concatenate([xr, xy + np.array([3.0, 0.5])])
    tri2 = np.concatenate([tr, tri + xr.shape[0]]).astype(np.int32)
    assert_parity(xy2, tri2, stages=False)


@pytest.mark.parametrize("s", [2, 3, 10, 33, 64, 200])
def test_regular_grid(s):
    res, _ = assert_parity(*synth.grid(s))
    assert res["P"] == (s - 1) ** 2


@pytest.mark.parametrize("s,seed", [(32, 1), (45, 7), (150, 3)])
def test_jittered_grid(s, seed):
    assert_parity(*synth.grid(s, 0.2, seed))


@pytest.mark.parametrize("n,seed", [(10, 1), (100, 2), (1000, 3), (5000, 4), (30000, 5), (200000, 6)])
def test_random_delaunay(n, seed):
    res, _ = assert_parity(*synth.random_delaunay(n, seed))
    if n >= 1000:
        assert res["n_tips"] > 0


def test_flip_walk_non_delaunay():
    rng = np.random.default_rng(0)
    for i, n in enumerate([50, 300, 2000]):
        xy, tri = synth.random_delaunay(n, 40 + i)
        assert_parity(xy, flip_walk(xy, tri, tri.shape[0] // 2, rng))


def test_shuffled_and_rotated_input():
    """Any triangle order / vertex rotation / orientation (worst case for the tile
    match: almost every twin is found through the global leftover hash)."""
    rng = np.random.default_rng(1)
    xy, tri = synth.random_delaunay(50000, 11)
    perm = rng.permutation(tri.shape[0])
    tri2 = tri[perm]
    rot = rng.integers(0, 3, size=tri2.shape[0])
    tri2 = np.stack([np.roll(t, r) for t, r in zip(tri2, rot)]).astype(np.int32)
    flip = rng.random(tri2.shape[0]) < 0.5
    tri2[flip] = tri2[flip][:, [0, 2, 1]]
    res, ref = assert_parity(xy, tri2)
    assert res["n_leftover"] > 0.9 * 3 * tri.shape[0]


def test_config1():
    res, ref = assert_parity(*synth.grid(32, 0.2, 1))
    assert res["n_tips"] == 0


@pytest.mark.slow
def test_config2_full():
    """BASELINE config 2 at full size: 1M random points (~2M triangles)."""
    xy, tri = synth.random_delaunay(1_000_000, 2)
    assert_parity(xy, tri, invariants=False)


@pytest.mark.slow
def test_config5_grid_full():
    """One config-5 regular grid at full size (s = 2000), closed form P = 1999^2."""
    xy, tri = synth.grid(2000)
    res, _ = assert_parity(xy, tri, stages=False, invariants=False)
    assert res["P"] == 3_996_001 and res["L"] == 15_984_004


def _grid_with_holes(s=60, seed=11):
    """Jittered grid minus the triangles with a vertex strictly inside three discs: four
    boundary loops (the outer one and three holes), polygons that touch the holes."""
    xy, tri = synth.grid(s, 0.2, seed)
    bad = np.zeros(tri.shape[0], bool)
    for cx, cy, r in ((0.25 * s, 0.26 * s, 0.10 * s), (0.67 * s, 0.37 * s, 0.085 * s), (0.5 * s, 0.76 * s, 0.12 * s)):
        bad |= (np.hypot(xy[:, 0] - cx, xy[:, 1] - cy) < r)[tri].any(axis=1)
    return xy, np.ascontiguousarray(tri[~bad])


def _wheels(k=300, seed=5):
    """k disjoint wheels (a centre vertex with 20-60 spokes each): rotation chains far
    longer than the 16 steps k_tile resolves in shared memory, so the label fixup walks
    them; several tiles."""
    rng = np.random.default_rng(seed)
    pts, tris, off = [], [], 0
    for w in range(k):
        n = int(rng.integers(20, 61))
        ang = np.sort(rng.random(n)) * 2 * np.pi
        rr = 1.0 + 0.4 * rng.random(n)
        c = np.array([3.0 * (w % 20), 3.0 * (w // 20)])
        pts.append(np.vstack([c, c + np.c_[rr * np.cos(ang), rr * np.sin(ang)]]))
        tris.append(np.array([[off, off + 1 + i, off + 1 + (i + 1) % n] for i in range(n)], np.int32))
        off += n + 1
    return np.vstack(pts), np.vstack(tris)


def test_mesh_with_holes():
    xy, tri = _grid_with_holes()
    res, ref = assert_parity(xy, tri)
    assert ref["B"] > 4 * 59  # outer boundary plus the three holes


def test_disconnected_components():
    xy1, tri1 = synth.grid(60, 0.2, 11)
    xy2, tri2 = synth.random_delaunay(5000, 12)
    xy = np.vstack([xy1, xy2 * 50.0 + np.array([100.0, 0.0])])
    tri = np.vstack([tri1, tri2 + xy1.shape[0]]).astype(np.int32)
    assert_parity(xy, tri)


def test_high_degree_wheels():
    xy, tri = _wheels()
    res, ref = assert_parity(xy, tri)
    assert res["n_deferred"] > 0


def _regions_case(name):
    if name == "square":
        return synth.fixture_square()
    if name == "fan":
        return synth.fixture_fan()
    if name == "tie":
        return synth.fixture_tie_lattice()
    if name == "grid":
        return synth.grid(64)
    if name == "jittered":
        return synth.grid(150, 0.2, 3)
    if name == "random":
        return synth.random_delaunay(200000, 6)
    if name == "holes":
        return _grid_with_holes()
    if name == "wheels":
        return _wheels()
    xy, tri = synth.random_delaunay(30000, 9)  # shuffled: the global leftover path
    return xy, np.ascontiguousarray(tri[np.random.default_rng(1).permutation(tri.shape[0])])


@pytest.mark.parametrize("name", ["square", "fan", "tie", "grid", "jittered", "random", "holes", "wheels", "shuffled"])
def test_triangle_polygons(name):
    """polylla_get_triangle_polygons against the oracle's flood
    definition, element by element (holes: several loops per piece -> the smallest)."""
    xy, tri = _regions_case(name)
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, regions=True)
    np.testing.assert_array_equal(res["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(ref))


@pytest.mark.parametrize("name", ["square", "fan", "tie", "grid", "jittered", "random", "holes", "wheels", "shuffled"])
def test_triangle_regions(name):
    """polylla_get_triangle_regions (NEXT-4, pre-repair Lepp partition) against the
    oracle's definition, element by element."""
    xy, tri = _regions_case(name)
    ref = oracle.run(xy, tri)
    res = gpu_run(xy, tri, regions=True)
    np.testing.assert_array_equal(res["region_of_tri"].cpu().numpy(), oracle.triangle_regions(ref))


def test_determinism_and_streams():
    xy, tri = synth.random_delaunay(20000, 8)
    a = gpu_run(xy, tri)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = gpu_run(xy, tri, stream=s)
    s.synchronize()
    for k in ("origin", "twin", "next", "offsets", "loops", "seeds"):
        assert torch.equal(a[k], b[k]), k


def test_concurrent_meshes_on_two_streams():
    """bench.py's batch path: independent meshes converted concurrently on two streams
    (own workspace and outputs each) give the same CSR as one at a time."""
    pp = _pp()
    meshes = [synth.grid(300, 0.2, 7), synth.grid(300), synth.random_delaunay(60000, 9), synth.grid(250, 0.2, 3)]
    ref = [gpu_run(xy, tri) for xy, tri in meshes]
    Vm = max(xy.shape[0] for xy, _ in meshes)
    Tm = max(tri.shape[0] for _, tri in meshes)
    lanes = []
    for _ in range(2):
        lanes.append(dict(stream=torch.cuda.Stream(), ws=pp.alloc_workspace(Vm, Tm), out=[]))
    dev = [(torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()) for xy, tri in meshes]
    torch.cuda.synchronize()
    for i, (xy_d, tri_d) in enumerate(dev):
        ln = lanes[i % 2]
        offs = torch.empty(Tm + 1, dtype=torch.int32, device="cuda")
        loops = torch.empty(3 * Tm, dtype=torch.int32, device="cuda")
        ctx = pp.build_halfedges(xy_d, tri_d, ln["ws"], ln["stream"])
        pp.label(ctx, ln["stream"])
        pp.generate(ctx, ln["stream"])
        pp.get_polygons(ctx, offs, loops, stream=ln["stream"])
        ln["out"].append((i, offs, loops))  # (a lane's next mesh reuses its workspace in stream order)
        pp.destroy(ctx)
    torch.cuda.synchronize()
    for ln in lanes:
        for i, offs, loops in ln["out"]:
            P, L = ref[i]["P"], ref[i]["L"]
            assert torch.equal(offs[:P + 1], ref[i]["offsets"]), i
            assert torch.equal(loops[:L], ref[i]["loops"]), i


def test_run_host_e2e_matches_oracle():
    """polylla_run_host (host buffers in, host buffers out) against the oracle."""
    pp = _pp()
    for xy, tri in (synth.random_delaunay(30000, 12), synth.grid(120, 0.2, 4)):
        ref = oracle.run(xy, tri)
        b = pp.run_host(xy, tri)
        assert b["H"] == ref["H"] and b["P"] == ref["P"]
        for k in ("origin", "twin", "next", "offsets", "loops"):
            np.testing.assert_array_equal(b[k].numpy(), ref[k], err_msg=k)


def _gpu_status(xy, tri, check=False):
    pp = _pp()
    with pytest.raises(pp.PolyllaError) as ei:
        gpu_run(np.asarray(xy, np.float64), np.asarray(tri, np.int32), check=check)
    return pp.STATUS[ei.value.code]


def _cross_tile_nonmanifold(two_pairs):
    """A jittered grid (T = 3,042 > one 2,048-triangle build tile) plus, at the end (tile 1),
    a triangle on an interior edge {a, b} of tile 0 -- the edge's third copy -- or
    (two_pairs) two triangles pairing on {a, b} inside tile 1 (copies three and four)."""
    xy, tri = synth.grid(40, 0.2, 5)
    a, b = int(tri[700, 0]), int(tri[700, 1])
    c = np.array([[1000.0, 1000.0], [-1000.0, -1000.0]])
    V = xy.shape[0]
    extra = [[a, b, V], [b, a, V + 1]] if two_pairs else [[a, b, V]]
    return np.vstack([xy, c]), np.vstack([tri, np.array(extra, np.int32)]).astype(np.int32)


@pytest.mark.parametrize("two_pairs", [False, True])
def test_cross_tile_nonmanifold_edge(two_pairs):
    """R20: copies of an edge paired inside one tile plus copies in another tile.  The
    oracle reports NON_MANIFOLD_EDGE; so does the GPU with polylla_check_manifold."""
    xy, tri = _cross_tile_nonmanifold(two_pairs)
    with pytest.raises(oracle.OracleError) as ei:
        oracle.run(xy, tri)
    assert oracle.STATUS[ei.value.code] == "NON_MANIFOLD_EDGE"
    assert _gpu_status(xy, tri, check=True) == "NON_MANIFOLD_EDGE"


def test_check_manifold_passes_valid_meshes():
    """The exact check raises nothing on valid meshes (shuffled input: every twin crosses
    tiles) and leaves the results bit-exact."""
    rng = np.random.default_rng(2)
    xy, tri = synth.random_delaunay(30000, 13)
    for t in (tri, np.ascontiguousarray(tri[rng.permutation(tri.shape[0])])):
        ref = oracle.run(xy, t)
        res = gpu_run(xy, t, check=True)
        np.testing.assert_array_equal(res["loops"].cpu().numpy(), ref["loops"])
        np.testing.assert_array_equal(res["next"].cpu().numpy(), ref["next"])


def test_error_kinds_match_oracle():
    sq_xy, _ = synth.fixture_square()
    cases = [
        (sq_xy, [[0, 1, 7]]),
        ([[0, 0], [1, 0], [2, 0]], [[0, 1, 2]]),
        (sq_xy, [[0, 1, 1]]),
        ([[0, 0], [1, 0], [0.5, 1], [0.5, -1], [0.5, 2]], [[0, 1, 2], [1, 0, 3], [0, 1, 4]]),
        ([[0, 0], [1, 0], [0.5, 1], [0.5, 2]], [[0, 1, 2], [0, 1, 3]]),
        ([[0, 0], [1, 0], [1, 1], [-1, 0], [-1, -1]], [[0, 1, 2], [0, 3, 4]]),
    ]
    for xy, tri in cases:
        with pytest.raises(oracle.OracleError) as ei:
            oracle.run(np.asarray(xy, np.float64), np.asarray(tri, np.int32))
        assert _gpu_status(xy, tri) == oracle.STATUS[ei.value.code]
        assert _gpu_status(xy, tri, check=True) == oracle.STATUS[ei.value.code]


def test_call_order_and_workspace_errors():
    pp = _pp()
    xy = torch.from_numpy(synth.fixture_square()[0]).cuda()
    tri = torch.from_numpy(synth.fixture_square()[1]).cuda()
    small = torch.empty(16, dtype=torch.uint8, device="cuda")
    with pytest.raises(pp.PolyllaError) as ei:
        pp.build_halfedges(xy, tri, small)
    assert pp.STATUS[ei.value.code] == "WORKSPACE"
    ws = pp.alloc_workspace(4, 2)
    ctx = pp.build_halfedges(xy, tri, ws)
    with pytest.raises(pp.PolyllaError) as ei:
        pp.generate(ctx)
    assert pp.STATUS[ei.value.code] == "CALL_ORDER"
    with pytest.raises(pp.PolyllaError) as ei:  # needs the polygon seeds of get_polygons
        pp.get_triangle_polygons(ctx, torch.empty(2, dtype=torch.int32, device="cuda"))
    assert pp.STATUS[ei.value.code] == "CALL_ORDER"
    pp.destroy(ctx)


@pytest.mark.slow
def test_config3_full():
    """BASELINE config 3 at full size (10M random points, ~20M triangles), the bench
    workload, in the launch configuration bench.py times: every array bit-exact."""
    xy, tri = synth.random_delaunay(10_000_000, 3)
    assert_parity(xy, tri, stages=False, invariants=False)


@pytest.mark.slow
def test_config3_triangle_polygons_areas():
    """Per-triangle polygon ids at the config-3 size, by properties that hold at any size
    (device-side): ids in [0, P), every polygon owns a triangle, and each polygon's loop
    area (shoelace over its CSR loop) equals the summed area of its triangles (rel 1e-9)."""
    xy, tri = synth.random_delaunay(10_000_000, 3)
    res = gpu_run(xy, tri, arrays=True, regions=True)
    P = res["P"]
    o = res["poly_of_tri"].long()
    assert int(o.min()) == 0 and int(o.max()) == P - 1
    xy_d = torch.from_numpy(xy).cuda()
    t = res["origin"][:3 * tri.shape[0]].long().view(-1, 3)
    a, b, c = xy_d[t[:, 0]], xy_d[t[:, 1]], xy_d[t[:, 2]]
    ta = (b[:, 0] - a[:, 0]) * (c[:, 1] - a[:, 1]) - (b[:, 1] - a[:, 1]) * (c[:, 0] - a[:, 0])
    tri_sum = torch.zeros(P, dtype=torch.float64, device="cuda").index_add_(0, o, ta)
    off = res["offsets"].long()
    lp = res["loops"].long()
    nxt = torch.arange(1, lp.numel() + 1, device="cuda")
    nxt[off[1:] - 1] = off[:-1]
    pe = torch.repeat_interleave(torch.arange(P, device="cuda"), off[1:] - off[:-1])
    base = xy_d[lp[off[:-1]]][pe]  # each loop relative to its first vertex (no cancellation)
    u, v = xy_d[lp] - base, xy_d[lp[nxt]] - base
    shoe = torch.zeros(P, dtype=torch.float64, device="cuda").index_add_(0, pe, u[:, 0] * v[:, 1] - v[:, 0] * u[:, 1])
    assert bool((tri_sum > 0).all())
    assert float(((shoe - tri_sum).abs() / tri_sum).max()) < 1e-9


@pytest.mark.slow
def test_config5_jittered_full():
    """A config-5 jittered mesh at full size (s = 2000, a = 0.2, seed 1000)."""
    xy, tri = synth.grid(2000, 0.2, 1000)
    assert_parity(xy, tri, stages=False, invariants=False)


def u32(t):
    """An int32 tensor of unsigned 32-bit half-edge ids / offsets (include/polylla.h) as int64."""
    return t.long() & 0xFFFFFFFF


def device_invariants(xy, tri, origin, twin, nxt, offsets, loops, seeds, chunk=1 << 26):
    """Invariants that hold at any size (north_star / SPEC.md L187-193), evaluated on the
    device with plain torch ops in chunks (test infrastructure).  Half-edge ids and
    offsets are read as unsigned (H may exceed 2^31, NEXT-3).  Returns P."""
    T = tri.shape[0]
    H = origin.numel()
    dev = origin.device
    for a in range(0, H, chunk):
        b = min(H, a + chunk)
        ids = torch.arange(a, b, device=dev)
        tw = u32(twin[a:b])
        assert torch.equal(u32(twin[tw]), ids) and not torch.any(tw == ids)     # twin involution
        assert torch.equal(origin[u32(nxt[a:b])], origin[tw])                    # origin(next e) = target(e)
    P = seeds.numel()
    off = u32(offsets)
    assert int(off[0]) == 0 and int(off[-1]) == loops.numel() and bool(torch.all(off[1:] > off[:-1]))
    sdall = u32(seeds)
    assert bool(torch.all(sdall[1:] > sdall[:-1])) and bool(torch.all(sdall < 3 * T))
    del sdall
    poly_area = 0.0
    xyd = xy.double()
    for a in range(0, P, chunk):
        b = min(P, a + chunk)
        sd = u32(seeds[a:b])
        o0, o1 = off[a:b], off[a + 1:b + 1]
        lens = o1 - o0
        assert torch.equal(loops[o0].long(), origin[sd].long())                 # loops start at origin[seed]
        # lock-step walk of the loops: each closes after exactly its length, never meets
        # next == twin, and never visits a half-edge below its seed (canonical = min)
        x = sd.clone()
        px = xyd[origin[x].long()]
        first = px.clone()
        area = torch.zeros(b - a, dtype=torch.float64, device=dev)
        for i in range(int(lens.max())):
            live = lens > i
            xi = x[live]
            assert torch.equal(origin[xi].long(), loops[o0[live] + i].long())
            assert not torch.any(nxt[xi] == twin[xi])
            assert bool(torch.all(xi >= sd[live]))
            x[live] = u32(nxt[xi])
            cur = px[live]
            nx_pt = torch.where((lens[live] > i + 1).unsqueeze(1), xyd[origin[x[live]].long()], first[live])
            area[live] += cur[:, 0] * nx_pt[:, 1] - nx_pt[:, 0] * cur[:, 1]
            px[live] = nx_pt
        assert torch.equal(x, sd)
        poly_area += 0.5 * float(area.sum())
    tri_area = 0.0
    for a in range(0, T, chunk):
        p = xyd[tri[a:a + chunk].long()]
        tri_area += 0.5 * float(((p[:, 1, 0] - p[:, 0, 0]) * (p[:, 2, 1] - p[:, 0, 1]) -
                                 (p[:, 1, 1] - p[:, 0, 1]) * (p[:, 2, 0] - p[:, 0, 0])).abs().sum())
    assert abs(poly_area - tri_area) <= 1e-9 * tri_area, (poly_area, tri_area)
    return P


@pytest.mark.slow
def test_config4_capacity_invariants():
    """BASELINE config 4 (256M vertices, 512M triangles, H = 1,535,872,002 < 2^31): the
    oracle cannot run at this size on the box, so the properties that hold at any size
    are checked on the device, reading the arrays in place in the workspace."""
    pp = _pp()
    xy, tri = synth.grid_device(16000, 0.2, 4)
    T = tri.shape[0]
    ws = pp.alloc_workspace(xy.shape[0], T)
    ctx = pp.build_halfedges(xy, tri, ws)
    pp.label(ctx)
    pp.generate(ctx)
    c = pp.get_counts(ctx)
    H, P, L = c["n_halfedges"], c["n_polygons"], c["n_loop_entries"]
    assert H == 1_535_872_002 and c["n_border"] == 4 * 15999
    offsets = torch.empty(T + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(3 * T, dtype=torch.int32, device="cuda")
    pp.get_polygons(ctx, offsets, loops)
    pp.get_counts(ctx)
    v = pp.get_views(ctx)
    view = lambda k, n: pp.view_tensor(ctx, v[k], n, torch.int32)  # noqa: E731
    got = device_invariants(xy, tri, view("origin", H), view("twin", H), view("next", H), offsets[:P + 1],
                            loops[:L], view("seeds", P))
    assert got == P
    pp.destroy(ctx)


def test_device_invariants_on_random_mesh():
    xy, tri = synth.random_delaunay(100_000, 21)
    res = gpu_run(xy, tri)
    P = device_invariants(torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda(), res["origin"], res["twin"],
                          res["next"], res["offsets"], res["loops"], res["seeds"], chunk=1 << 14)
    assert P == res["P"]


def test_cuda_graph_replay_matches_eager():
    pp = _pp()
    xy, tri = synth.random_delaunay(50_000, 31)
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    ref = gpu_run(xy, tri)
    T = tri.shape[0]
    ws = pp.alloc_workspace(xy.shape[0], T)
    offsets = torch.empty(T + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(3 * T, dtype=torch.int32, device="cuda")
    g = pp.GraphStep(xd, td, ws, offsets, loops)
    for _ in range(3):
        offsets.fill_(-1)
        loops.fill_(-1)
        g.replay()
        g.stream.synchronize()
        P, L = ref["P"], ref["L"]
        assert torch.equal(offsets[:P + 1], ref["offsets"]) and torch.equal(loops[:L], ref["loops"])


def test_host_pipeline_matches_oracle():
    """HostPipeline (pinned host in/out, copies overlapped across meshes) against the oracle."""
    pp = _pp()
    meshes = [synth.random_delaunay(20_000, 50 + i) for i in range(3)] + [synth.grid(90, 0.2, 9)]
    V = max(m[0].shape[0] for m in meshes)
    T = max(m[1].shape[0] for m in meshes)
    pipe = pp.HostPipeline(V, T)
    inputs = [(torch.from_numpy(x).pin_memory(), torch.from_numpy(t).pin_memory()) for x, t in meshes]
    outs = [pp.alloc_host_outputs(T) for _ in meshes]
    counts = pipe.run(inputs, outs)
    for (x, t), o, c in zip(meshes, outs, counts):
        ref = oracle.run(x, t)
        P, L, H = c["n_polygons"], c["n_loop_entries"], c["n_halfedges"]
        assert (P, L, H) == (ref["P"], ref["L"], ref["H"])
        np.testing.assert_array_equal(o["offsets"][:P + 1].numpy(), ref["offsets"])
        np.testing.assert_array_equal(o["loops"][:L].numpy(), ref["loops"])
        for k in ("origin", "twin", "next"):
            np.testing.assert_array_equal(o[k][:H].numpy(), ref[k], err_msg=k)
