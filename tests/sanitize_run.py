"""Small conversions for compute-sanitizer runs: fixtures, a jittered grid, a random mesh
(multi-tile), a shuffled mesh (global leftover path).  Exits non-zero on any mismatch with
the oracle."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2403_14723_b200 import polylla as pp  # noqa: E402

cases = [synth.fixture_square(), synth.fixture_fan(), synth.fixture_tie_lattice(), synth.grid(32, 0.2, 1),
         synth.random_delaunay(6000, 5)]
xy, tri = synth.random_delaunay(3000, 6)
cases.append((xy, tri[np.random.default_rng(0).permutation(tri.shape[0])]))
for xy, tri in cases:
    r = pp.run(torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda(), prev=True, regions=True)
    o = oracle.run(xy, tri)
    for k in ("origin", "twin", "next", "prev"):
        assert np.array_equal(r[k].cpu().numpy(), o[k]), k
    assert np.array_equal(r["loops"].cpu().numpy(), o["loops"])
    assert np.array_equal(r["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(o))
# the bounded layout (NEXT-3), the paper ablation (NEXT-2), the non-manifold check, the
# pre-repair regions and run_host (NEXT-1) on one multi-tile mesh
xy, tri = synth.random_delaunay(6000, 7)
o = oracle.run(xy, tri)
xd, td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
B = o["H"] - 3 * tri.shape[0]
for paper in (False, True):
    ws = pp.alloc_workspace(xy.shape[0], tri.shape[0], max_border=B, staging=False)
    ctx = pp.build_halfedges(xd, td, ws, max_border=B, staging=False)
    pp.check_manifold(ctx)
    if paper:
        pp.label_generate_paper(ctx)
    else:
        pp.label(ctx)
        reg = torch.empty(tri.shape[0], dtype=torch.int32, device="cuda")
        pp.get_triangle_regions(ctx, reg)
        pp.generate(ctx)
    c = pp.get_counts(ctx)
    off = torch.empty(c["n_polygons"] + 1, dtype=torch.int32, device="cuda")
    lp = torch.empty(c["n_loop_entries"], dtype=torch.int32, device="cuda")
    pp.get_polygons(ctx, off, lp)
    assert pp.get_counts(ctx)["status"] == 0
    assert np.array_equal(lp.cpu().numpy(), o["loops"]) and np.array_equal(off.cpu().numpy(), o["offsets"])
    pp.destroy(ctx)
# grid tiling (row-stride hint): a jittered grid with partial tiles, regions included
gx, gt = synth.grid(150, 0.2, 9)
go = oracle.run(gx, gt)
gr = pp.run(torch.from_numpy(gx).cuda(), torch.from_numpy(gt).cuda(), row_stride=2 * 149, prev=True, regions=True)
for k in ("origin", "twin", "next", "prev"):
    assert np.array_equal(gr[k].cpu().numpy(), go[k]), k
assert np.array_equal(gr["poly_of_tri"].cpu().numpy(), oracle.triangle_polygons(go))
# sorted tiling (POLYLLA_BUILD_SORT) on a shuffled mesh
sx, st = synth.random_delaunay(5000, 31)
st = np.ascontiguousarray(st[np.random.default_rng(2).permutation(st.shape[0])])
so = oracle.run(sx, st)
sr = pp.run(torch.from_numpy(sx).cuda(), torch.from_numpy(st).cuda(), sort=True, prev=True, regions=True)
for k in ("origin", "twin", "next", "prev"):
    assert np.array_equal(sr[k].cpu().numpy(), so[k]), k
assert np.array_equal(sr["loops"].cpu().numpy(), so["loops"])
h = pp.run_host(xy, tri)
assert np.array_equal(h["loops"].numpy(), o["loops"]) and np.array_equal(h["next"].numpy(), o["next"])
print("sanitize cases ok", len(cases) + 5)
