import sys; sys.path.insert(0,'.')
import torch, synth
from paper_2403_14723_b200 import polylla as pp
xy,tri = synth.grid(10)
r = pp.run(torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda())
print("ok", r["P"])
