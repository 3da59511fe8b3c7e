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
print("sanitize cases ok", len(cases))
