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


def test_determinism_and_streams():
    xy, tri = synth.random_delaunay(20000, 8)
    a = gpu_run(xy, tri)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = gpu_run(xy, tri, stream=s)
    s.synchronize()
    for k in ("origin", "twin", "next", "offsets", "loops", "seeds"):
        assert torch.equal(a[k], b[k]), k


def test_run_host_e2e_matches_device():
    pp = _pp()
    xy, tri = synth.random_delaunay(30000, 12)
    a = gpu_run(xy, tri)
    b = pp.run_host(xy, tri)
    for k in ("origin", "twin", "next", "offsets", "loops"):
        np.testing.assert_array_equal(a[k].cpu().numpy(), b[k].numpy(), err_msg=k)


def _gpu_status(xy, tri):
    pp = _pp()
    with pytest.raises(pp.PolyllaError) as ei:
        gpu_run(np.asarray(xy, np.float64), np.asarray(tri, np.int32))
    return pp.STATUS[ei.value.code]


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
    pp.destroy(ctx)
