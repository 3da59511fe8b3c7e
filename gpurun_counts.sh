python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
import synth
from paper_2403_14723_b200 import polylla as pp
for name, (xy, tri) in [("c3", synth.random_delaunay(10_000_000, 3)), ("c5j", synth.grid(2000, 0.2, 1000)), ("c5r", synth.grid(2000))]:
    r = pp.run(torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda(), arrays=False)
    T = tri.shape[0]
    print(name, "T", T, {k: (r[k], round(r[k] / (3 * T), 4)) for k in ("n_leftover", "n_deferred", "n_seed_deferred", "n_tips", "P")})
PY
