"""Diagnostics: per-phase cycle breakdown of k_tile (builds a POLYLLA_PHASE_TIMING variant
of the library under /tmp, runs config 3 a few times, prints average cycles per tile)."""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa
import torch  # noqa

so = "/tmp/libpolylla_phase%s.so" % os.getpid()
# POLYLLA_SRC: another source tree (A/B against an older commit: git archive ... | tar -x -C DIR)
SRC = os.environ.get("POLYLLA_SRC", ROOT)
csrc = os.path.join(SRC, "paper_2403_14723_b200", "csrc")
cu = [os.path.join(csrc, f) for f in sorted(os.listdir(csrc)) if f.endswith(".cu")]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
                "-DPOLYLLA_PHASE_TIMING", "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-I",
                os.path.join(SRC, "include"), "-o", so, *cu], check=True)
from paper_2403_14723_b200 import polylla as pp  # noqa
pp.LIB_PATH = so
L = pp.lib()
L.polylla_debug_phase_cycles.argtypes = [ctypes.c_void_p, ctypes.c_int]
import synth  # noqa
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
n = {2: 1_000_000, 3: 10_000_000}[cfg]
xy, tri = synth.random_delaunay(n, cfg)
xy_d, tri_d = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
ws = pp.alloc_workspace(xy.shape[0], tri.shape[0])
buf = np.zeros(16, np.uint64)
reps = 5
for r in range(reps + 1):
    if r == 1:
        torch.cuda.synchronize()
        L.polylla_debug_phase_cycles(buf.ctypes.data, 1)
    ctx = pp.build_halfedges(xy_d, tri_d, ws)
    pp.destroy(ctx)
torch.cuda.synchronize()
L.polylla_debug_phase_cycles(buf.ctypes.data, 0)
tiles = (tri.shape[0] + 2047) // 2048
names = ["P0 clear", "P1 orient/lcode", "P2 hash", "P3 succ/out", "P4a jump", "P4b label/next", "P5+P6 lists/seeds",
         "out (word stores)"]
tot = buf[:8].sum()
for i, nme in enumerate(names):
    print(f"{nme:18s} {buf[i] / (reps * tiles):10.0f} cycles/tile  {100 * buf[i] / tot:5.1f}%")
print("total", buf[:8].sum() / (reps * tiles), "cycles/tile")
