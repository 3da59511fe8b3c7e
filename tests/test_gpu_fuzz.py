"""Randomised cross-checks against the CPU oracle: mesh kind and size, triangle order,
per-triangle orientation, build tiling (contiguous, grid with a valid row stride, sorted)
and workspace layout (worst case or bounded border, with or without staging) drawn from a
seeded generator; every output element compared (origin/twin/next/prev, seeds, CSR, the
stage bit-vectors, per-triangle polygon ids)."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import bits_to_bool

pytestmark = pytest.mark.gpu


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = rng.choice(["random", "grid", "jittered"])
    if kind == "random":
        xy, tri = synth.random_delaunay(int(rng.integers(20, 30000)), int(rng.integers(1, 10**6)))
        R = 0
    else:
        s = int(rng.integers(3, 140))
        xy, tri = synth.grid(s, 0.2 if kind == "jittered" else 0.0, int(rng.integers(0, 1000)))
        R = 2 * (s - 1)
    T = tri.shape[0]
    order = rng.choice(["as-is", "shuffled", "reversed"])
    if order == "shuffled":
        tri = tri[rng.permutation(T)]
        R = 0  # (no longer row-major)
    elif order == "reversed":
        tri = tri[::-1]
        R = 0
    flip = rng.random(T) < 0.5  # random orientation: CW triangles are re-oriented (R10)
    tri = tri.copy()
    tri[flip, 1], tri[flip, 2] = tri[flip, 2].copy(), tri[flip, 1].copy()
    tiling = rng.choice(["contiguous", "grid", "sorted"]) if R else rng.choice(["contiguous", "sorted"])
    return kind, order, tiling, xy, np.ascontiguousarray(tri, dtype=np.int32), R, bool(rng.random() < 0.5)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_vs_oracle(seed):
    from paper_2403_14723_b200 import polylla as pp
    kind, order, tiling, xy, tri, R, bounded = _case(seed)
    T = tri.shape[0]
    ref = oracle.run(xy, tri)
    H, P, L = ref["H"], ref["P"], ref["L"]
    B = H - 3 * T
    kw = dict(row_stride=R if tiling == "grid" else 0, sort=tiling == "sorted")
    if bounded:
        kw.update(max_border=B, staging=False)
    xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
    ws = pp.alloc_workspace(xy.shape[0], T, **kw)
    ctx = pp.build_halfedges(xd, td, ws, **kw)
    pp.label(ctx)
    pp.generate(ctx)
    c = pp.get_counts(ctx)
    assert (c["n_halfedges"], c["n_polygons"], c["n_loop_entries"], c["n_flips"]) == (H, P, L, ref["flips"]), \
        (kind, order, tiling, bounded)
    out = {k: torch.empty(n, dtype=torch.int32, device="cuda")
           for k, n in (("offsets", P + 1), ("loops", L), ("origin", H), ("twin", H), ("next", H), ("prev", H))}
    pp.get_polygons(ctx, out["offsets"], out["loops"], origin=out["origin"], twin=out["twin"], next=out["next"],
                    prev=out["prev"])
    pot = torch.empty(T, dtype=torch.int32, device="cuda")
    pp.get_triangle_polygons(ctx, pot)
    assert pp.get_counts(ctx)["status"] == 0
    for k in ("offsets", "loops", "origin", "twin", "next", "prev"):
        np.testing.assert_array_equal(out[k].cpu().numpy(), ref[k], err_msg=f"{k} {kind} {order} {tiling}")
    v = pp.get_views(ctx)
    np.testing.assert_array_equal(pp.view_tensor(ctx, v["seeds"], P, torch.int32).cpu().numpy(), ref["seeds"])
    nw = (3 * T + 31) // 32
    for k, r in (("frontier0", "frontier0"), ("frontier1", "frontier1")):
        got = bits_to_bool(pp.view_tensor(ctx, v[k], nw, torch.int32).clone(), 3 * T)
        np.testing.assert_array_equal(got, ref[r][:3 * T].astype(bool), err_msg=f"{k} {kind} {order} {tiling}")
    np.testing.assert_array_equal(pot.cpu().numpy(), oracle.triangle_polygons(ref))
    pp.destroy(ctx)
