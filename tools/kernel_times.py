"""Per-kernel-group medians over repeated eager steps (library CUDA events), plus the
graph-replayed step time -- a steadier A/B measure than bench.py's means.
usage: python tools/kernel_times.py [config=3] [reps=40] [lib ...]"""
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
libs = sys.argv[3:] or [None]
if cfg == 4:
    xy_d, tri_d = synth.grid_device(16000, 0.2, 4)
elif cfg == 5:
    xy, tri = synth.grid(2000, 0.2, 1000)
else:
    xy, tri = synth.random_delaunay({2: 1_000_000, 3: 10_000_000}[cfg], cfg)
if cfg != 4:
    xy_d, tri_d = torch.from_numpy(xy).cuda(), torch.from_numpy(tri).cuda()
V, T = xy_d.shape[0], tri_d.shape[0]
# POLYLLA_ROWS=1: grid configs (4, 5) pass their row stride 2(s-1) (grid tiling)
R = {4: 2 * 15999, 5: 2 * 1999}.get(cfg, 0) if os.environ.get("POLYLLA_ROWS") == "1" else 0
import importlib  # noqa: E402

for lib in libs:
    if lib:
        os.environ["POLYLLA_LIB"] = lib
    import paper_2403_14723_b200.polylla as pp
    pp = importlib.reload(pp)
    ws = pp.alloc_workspace(V, T, row_stride=R)
    offs = torch.empty(T + 1, dtype=torch.int32, device="cuda")
    loops = torch.empty(3 * T, dtype=torch.int32, device="cuda")
    s = torch.cuda.Stream()

    paper = os.environ.get("POLYLLA_PAPER") == "1"  # the paper's kernel sequence (NEXT-2 ablation)

    def step():
        ctx = pp.build_halfedges(xy_d, tri_d, ws, s, row_stride=R)
        if paper:
            pp.label_generate_paper(ctx, s)
        else:
            pp.label(ctx, s)
            pp.generate(ctx, s)
        pp.get_polygons(ctx, offs, loops, stream=s)
        pp.destroy(ctx)

    for _ in range(5):
        step()
    torch.cuda.synchronize()
    pp.profile_enable(True)
    per = {}
    for _ in range(reps):
        step()
        for k, (ms, _) in pp.profile_read().items():
            per.setdefault(k, []).append(ms)
    pp.profile_enable(False)
    g = pp.GraphStep(xy_d, tri_d, ws, offs, loops, s, paper=paper, row_stride=R)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(reps):
        e0.record(s)
        g.replay()
        e1.record(s)
        e1.synchronize()
        times.append(e0.elapsed_time(e1))
    med = {k: statistics.median(v) for k, v in per.items()}
    ctx = pp.build_halfedges(xy_d, tri_d, ws, s, row_stride=R)
    if paper:
        pp.label_generate_paper(ctx, s)
    else:
        pp.label(ctx, s)
        pp.generate(ctx, s)
    cn = pp.get_counts(ctx, s)
    pp.destroy(ctx)
    print("  counts: " + " ".join(f"{k}={cn[k]}" for k in ("n_leftover", "n_deferred", "n_seed_deferred", "n_tips",
                                                            "n_exact") if k in cn), flush=True)
    print(f"{os.path.basename(lib or pp.LIB_PATH)} cfg{cfg}: step(graph) median {statistics.median(times):.3f} ms  "
          f"min {min(times):.3f}  | " + " ".join(f"{k}={v:.3f}" for k, v in med.items()), flush=True)
    del g, ws, offs, loops
    torch.cuda.empty_cache()
