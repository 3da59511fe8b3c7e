import sys; sys.path.insert(0,'.')
import numpy as np, torch, synth, oracle
from paper_2403_14723_b200 import polylla as pp
xy,tri = synth.grid(int(sys.argv[1]) if len(sys.argv)>1 else 64)
T=tri.shape[0]
ws = pp.alloc_workspace(xy.shape[0], T)
xd,td = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
ctx = pp.build_halfedges(xd, td, ws); pp.label(ctx); pp.generate(ctx)
c = pp.get_counts(ctx, check=False); print(c)
v = pp.get_views(ctx)
ref = oracle.run(xy, tri)
def bits(off, n): 
    w = pp.view_tensor(ctx, off, (3*T+31)//32, torch.int32).cpu().numpy().view(np.uint8)
    return np.unpackbits(w, bitorder='little')[:n].astype(bool)
for k in ("frontier0","frontier1","seed_bits"):
    g = bits(v[k], 3*T); r = {"frontier0": ref["frontier0"][:3*T].astype(bool), "frontier1": ref["frontier1"][:3*T].astype(bool)}.get(k)
    if r is None: r = np.zeros(3*T,bool); r[ref["seeds0"]] = True
    print(k, "mismatch", int((g!=r).sum()), np.nonzero(g!=r)[0][:10])
H = c["n_halfedges"]
nx = pp.view_tensor(ctx, v["next"], H, torch.int32).cpu().numpy()
print("next mismatch", int((nx != ref["next"]).sum()), np.nonzero(nx != ref["next"])[0][:10])
