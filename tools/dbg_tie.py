import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch, synth
from paper_2403_14723_b200 import polylla as pp
pp.set_library(sys.argv[1])
xy, tri = synth.fixture_tie_lattice()
xy_d, tri_d = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
ws = pp.alloc_workspace(xy.shape[0], tri.shape[0])
s = torch.cuda.current_stream()
for name, f in [("build", lambda: pp.build_halfedges(xy_d, tri_d, ws, s))]:
    try:
        ctx = f(); torch.cuda.synchronize(); print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", repr(e)[:200], flush=True); sys.exit()
for name, f in [("label", lambda: pp.label(ctx, s)), ("generate", lambda: pp.generate(ctx, s))]:
    try:
        f(); torch.cuda.synchronize(); print(name, "ok", flush=True)
    except Exception as e:
        print(name, "FAIL", repr(e)[:200], flush=True); sys.exit()
try:
    print(pp.get_counts(ctx, s))
except Exception as e:
    print("counts FAIL", repr(e)[:300])
