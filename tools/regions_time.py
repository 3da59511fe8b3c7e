"""Time polylla_get_triangle_polygons (NEXT-4) on config 3 next to the step it follows:
median of CUDA-event times over repeated calls on the launching stream."""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2403_14723_b200 import polylla as pp  # noqa: E402

xy, tri = synth.random_delaunay(10_000_000, 3)
xy_d, tri_d = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
T = tri.shape[0]
ws = pp.alloc_workspace(xy.shape[0], T)
offs = torch.empty(T + 1, dtype=torch.int32, device="cuda")
loops = torch.empty(3 * T, dtype=torch.int32, device="cuda")
out = torch.empty(T, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
ts = []
for r in range(23):
    ctx = pp.build_halfedges(xy_d, tri_d, ws, s)
    pp.label(ctx, s)
    pp.generate(ctx, s)
    pp.get_polygons(ctx, offs, loops, stream=s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    pp.get_triangle_polygons(ctx, out, s)
    b.record(s)
    s.synchronize()
    if r >= 3:
        ts.append(a.elapsed_time(b))
    pp.destroy(ctx)
P = int(out.max().item()) + 1
print(f"get_triangle_polygons cfg3: T={T} P={P} median {statistics.median(ts):.3f} ms  min {min(ts):.3f}")
