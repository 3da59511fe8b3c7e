#!/usr/bin/env python
"""Benchmark of the B200 Polylla core (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]

A "step" is one pass of the whole hot path over one
mesh: polylla_build_halfedges -> polylla_label -> polylla_generate ->
polylla_get_polygons (CSR), inputs resident in HBM, no host sync inside the step.
Default workload: BASELINE config 3 (10M random points, Delaunay, ~20M triangles) --
the mesh the north_star's roofline target is stated on; its inputs (400 MB) and
working set (~1.7 GB) exceed the 126 MB L2, so no flush is needed between steps.

value      : input triangles/s, kernel-only, whole job (sum over ranks / max time)
e2e        : the same through polylla_run_host with pinned HOST buffers (H2D of xy+tri,
             kernels, D2H of CSR + origin/twin/next), CUDA events on the stream
roofline   : dominant kernel group, algorithmic bytes / its live CUDA-event time
cpu_baseline: the CPU oracle (oracle/, 1 thread) on a bounded sample, rank 0 at N=1
--impl reference: the oracle as the reference arm (each step a bounded sample).
Under torchrun (N > 1) every rank converts its own mesh (weak scaling, no collective
on the data path); the max device time over ranks is all-reduced through NCCL.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "input triangles/sec (kernel-only pipeline build->label->generate->CSR, 1 mesh per GPU)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=3, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def dist_setup():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return ws, rank, local


def workload(cfg: int, rank: int):
    """Synthetic input of BASELINE config `cfg` (recipes: DESIGN.md 'Input recipe')."""
    if cfg == 1:
        xy, tri = synth.grid(32, 0.2, 1)
        name = "config1: jittered 32x32 grid (a=0.2), 1 mesh"
    elif cfg == 2:
        xy, tri = synth.random_delaunay(1_000_000, 2 + 1000 * rank)
        name = "config2: 1M random points, Delaunay (Morton-ordered triangles), 1 mesh per GPU"
    elif cfg == 3:
        xy, tri = synth.random_delaunay(10_000_000, 3 + 1000 * rank)
        name = "config3: 10M random points, Delaunay (Morton-ordered triangles), 1 mesh per GPU"
    elif cfg == 4:
        xy, tri = synth.grid(16000, 0.2, 4)
        name = "config4: jittered 16000x16000 grid (256M vertices), 1 mesh per GPU"
    else:
        xy, tri = synth.grid(2000, 0.2 if rank % 2 == 0 else 0.0, 1000 + rank)
        name = "config5-slice: one 4M-vertex grid per GPU (jittered on even ranks, regular on odd)"
    return name, xy, tri


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    except Exception:
        return 6650.0, "fallback 6.65 TB/s from B200_PROFILING.md (MEASURED_PEAKS.json absent)"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.stop_ev = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        nv = self.nv
        names = {
            "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
            "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
            "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
        }
        while not self.stop_ev.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for k, v in names.items():
                    if r & v and k != "gpu_idle":
                        self.reasons.add(k)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop_ev.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def alg_bytes(T, V, P, L):
    """Algorithmic bytes: the method's compulsory HBM traffic."""
    return {
        "pipeline": 60 * T + 16 * V + 12 * L + 4 * P,
        # tri in + xy once + origin out + twin out + Lcode out
        "k_build_tile": 12 * T + 16 * V + 12 * T + 12 * T + T,
        # twin in + Lcode in + next out + F0/F1/S bit-vectors out
        "k_label_rewire": 12 * T + T + 12 * T + 3 * (3 * T) // 8,
        # S + F1 bits in, next re-read along the loops (L), canonical bits + len out
        "k_seed_walk": 2 * (3 * T) // 8 + 4 * L + (3 * T) // 8 + 4 * P,
        # seeds + offsets in, next + origin along the loops, loops + offsets out
        "k_extract": 4 * P + 4 * (P + 1) + 8 * L + 4 * L + 4 * (P + 1),
    }


def ncu_traffic(kernel: str, cfg: int):
    """dram__bytes_read+write per launch of `kernel` from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"config{cfg}", {}).get(kernel)
    except Exception:
        return None


def cpu_oracle_baseline(xy, tri, budget_s=30.0):
    """Time the CPU oracle on a bounded sample of the workload (rank 0, N = 1)."""
    import oracle
    T = tri.shape[0]
    if T <= 25_000_000:
        sample_xy, sample_tri, what = xy, tri, f"the full bench mesh ({T} triangles), 1 run"
    else:
        sample_xy, sample_tri = synth.random_delaunay(2_000_000, 99)
        what = f"a 2M-point random Delaunay mesh of the same recipe ({sample_tri.shape[0]} triangles), 1 run"
    t0 = time.perf_counter()
    o = oracle.run(sample_xy, sample_tri)
    dt = time.perf_counter() - t0
    return {"value": sample_tri.shape[0] / dt, "unit": "triangles/s", "cores": 1, "kind": "oracle",
            "sample": what, "seconds": dt, "phases_s": o["times"]}


def reference_arm(args, ws, rank):
    """--impl reference: the CPU oracle, unmodified, as the reference arm."""
    if rank != 0:
        return
    import oracle
    steps, warm = args.steps, args.warmup
    # calibrate: oracle throughput on a small mesh of the same recipe
    cxy, ctri = synth.random_delaunay(100_000, 7)
    t0 = time.perf_counter()
    oracle.run(cxy, ctri)
    rate = ctri.shape[0] / (time.perf_counter() - t0)
    budget = 150.0 / max(1, steps + warm)  # seconds per step so the run ends in ~2.5 min
    n = int(min(10_000_000, max(2_000, 0.5 * rate * budget)))
    sxy, stri = synth.random_delaunay(n, 3)
    for _ in range(warm):
        oracle.run(sxy, stri)
    t0 = time.perf_counter()
    for _ in range(steps):
        oracle.run(sxy, stri)
    dt = time.perf_counter() - t0
    T = stri.shape[0]
    v = T * steps / dt
    what = f"{n}-point random Delaunay mesh (config-{args.config} recipe, {T} triangles) per step"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "triangles/s", "n_gpus": ws,
        "steps": steps, "warmup": warm, "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64/i32", "data": "synthetic",
        "config": {"workload": what},
        "cpu_baseline": {"value": v, "unit": "triangles/s", "cores": 1, "kind": "oracle", "sample": what},
        "e2e": {"value": v, "unit": "triangles/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_setup()
    if args.impl == "reference":
        reference_arm(args, ws, rank)
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    from paper_2403_14723_b200 import polylla as pp

    dev = torch.device("cuda", local if ws > 1 else 0)
    name, xy_np, tri_np = workload(args.config, rank)
    V, T = xy_np.shape[0], tri_np.shape[0]
    xy = torch.from_numpy(xy_np).to(dev)
    tri = torch.from_numpy(tri_np).to(dev)
    wsp = pp.alloc_workspace(V, T, dev)
    offsets = torch.empty(T + 1, dtype=torch.int32, device=dev)
    loops = torch.empty(3 * T, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(device=dev)
    launches = [0]

    def step():
        ctx = pp.build_halfedges(xy, tri, wsp, stream)
        pp.label(ctx, stream)
        pp.generate(ctx, stream)
        pp.get_polygons(ctx, offsets, loops, stream=stream)
        launches[0] = pp.launch_count(ctx)
        return ctx

    # correctness gate + counts
    ctx = step()
    counts = pp.get_counts(ctx, stream)
    pp.destroy(ctx)
    P, L = counts["n_polygons"], counts["n_loop_entries"]

    for _ in range(args.warmup):
        pp.destroy(step())
    torch.cuda.synchronize(dev)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local if ws > 1 else 0) as clk:
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            pp.destroy(step())
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    if ws > 1:
        dist.barrier()
    ms_total = ev0.elapsed_time(ev1)
    t_max = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    tris = torch.tensor([float(T)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        dist.all_reduce(tris, op=dist.ReduceOp.SUM)
    ms_total = float(t_max.item())
    ms_step = ms_total / args.steps
    value = float(tris.item()) * args.steps / (ms_total / 1e3)
    ctx = step()
    final = pp.get_counts(ctx, stream)
    pp.destroy(ctx)
    assert final["status"] == 0 and final["n_polygons"] == P

    # ---- live per-kernel times (CUDA events recorded by the library on `stream`)
    pp.profile_enable(True)
    prof_steps = max(5, min(args.steps, 50))
    for _ in range(prof_steps):
        pp.destroy(step())
    prof = pp.profile_read()
    pp.profile_enable(False)
    per_launch = {k: ms / cnt for k, (ms, cnt) in prof.items()}
    prof_step_ms = sum(ms for ms, _ in prof.values()) / prof_steps
    ab = alg_bytes(T, V, P, L)
    peak, peak_src = load_peaks()
    top = max((k for k in per_launch if k in ab), key=lambda k: per_launch[k])
    achieved = ab[top] / (per_launch[top] * 1e-3) / 1e9
    traffic = ncu_traffic(top, args.config)
    roof = {"bound": "hbm", "kernel": top, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "alg_bytes_per_launch": ab[top],
            "kernel_ms": per_launch[top], "share_of_step": per_launch[top] / prof_step_ms, "peak_source": peak_src}
    pipe_gbs = ab["pipeline"] / (ms_step * 1e-3) / 1e9
    pipeline_roof = {"alg_bytes_per_step": ab["pipeline"], "achieved": pipe_gbs, "peak": peak,
                     "frac": pipe_gbs / peak, "frac_of_8TBs_nominal": pipe_gbs / 8000.0}

    # ---- end to end through polylla_run_host with pinned host buffers
    e2e = None
    if not args.no_e2e:
        xy_h = torch.from_numpy(xy_np).pin_memory()
        tri_h = torch.from_numpy(tri_np).pin_memory()
        outs = pp.alloc_host_outputs(T, arrays=True, pin=True)
        xy_hn, tri_hn = xy_h.numpy(), tri_h.numpy()
        for _ in range(2):
            r = pp.run_host(xy_hn, tri_hn, wsp, pinned=outs, stream=stream)
        torch.cuda.synchronize(dev)
        if ws > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            r = pp.run_host(xy_hn, tri_hn, wsp, pinned=outs, stream=stream)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        et = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e_ms = float(et.item()) / args.e2e_steps
        H = r["H"]
        e2e = {"value": float(tris.item()) / (e_ms / 1e3), "unit": "triangles/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": 16 * V + 12 * T, "d2h_bytes_per_step": 4 * (P + 1) + 4 * L + 3 * 4 * H,
               "api": "polylla_run_host (pinned host in/out; CSR + origin/twin/next returned)"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(xy_np, tri_np)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": "triangles/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64/i32", "data": "synthetic",
            "config": {"workload": name, "V": V, "T": T, "P": P, "L": L, "H": counts["n_halfedges"],
                       "tips": counts["n_tips"], "leftover_halfedges": counts["n_leftover"],
                       "l2": "no flush: inputs 16V+12T = %.0f MB and working set > 126 MB L2" %
                             ((16 * V + 12 * T) / 1e6)},
            "polygons_per_s": P * ws * args.steps / (ms_total / 1e3),
            "roofline": roof, "pipeline_roofline": pipeline_roof,
            "kernels_ms_per_step": {k: ms / prof_steps for k, (ms, _) in prof.items()},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches[0] * args.steps,
            "clocks": clk.summary(),
        }
        print(json.dumps(out), flush=True)
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
