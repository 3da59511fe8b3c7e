"""Compile-time variants of libpolylla.so for the schedule-independence and fallback-path
tests (results must not depend on the block -> tile schedule, the
block sizes or which path -- in-tile or global -- finishes a half-edge).

Each variant is the same sources built with extra -D flags into
paper_2403_14723_b200/variants/libpolylla_<name>.so (rebuilt when a source is newer):

  rev       tiles run in reverse block order (k_tile, leftover match, border ranking,
            label fixup, emission); 4 pointer-jumping rounds in k_tile
  threads   other block sizes for every global kernel, 4-word bit chunks; a k_tile hash
            of 4,104 slots (load 0.75: long probe runs, wrap-around at the table's end)
  tile384   k_tile with 384 threads (6 triangle iterations per thread), no pointer
            jumping (rotation chains resolved by hops only)
  fallback  a 64-entry k_emit queue (every tile takes the dense-tile branch) and an
            in-tile loop-walk bound of 3 (almost every seed goes to the global walk); repair
            rotations above degree 4 walked per incoming frontier half-edge
"""
from __future__ import annotations

import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2403_14723_b200")
OUT = os.path.join(PKG, "variants")

VARIANTS = {
    "rev": ["-DPOLYLLA_REVERSE_TILES", "-DPOLYLLA_TILE_JUMPS=4"],
    "threads": ["-DPOLYLLA_FIX_THREADS=128", "-DPOLYLLA_SEED_THREADS=128", "-DPOLYLLA_EMIT_THREADS=256",
                "-DPOLYLLA_REPAIR_THREADS=256", "-DPOLYLLA_LEFT_THREADS=128", "-DPOLYLLA_BIT_CHUNK=4",
                "-DPOLYLLA_UF_THREADS=256", "-DPOLYLLA_TILE_SLOTS=4104"],
    "tile384": ["-DPOLYLLA_TILE_THREADS=384", "-DPOLYLLA_TILE_JUMPS=0"],
    "fallback": ["-DPOLYLLA_EMIT_Q=64", "-DPOLYLLA_P6_MAXLEN=3", "-DPOLYLLA_ROT_MAX=4"],
}


def _sources():
    csrc = os.path.join(PKG, "csrc")
    cu = sorted(os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith(".cu"))
    hdr = [os.path.join(ROOT, "include", "polylla.h")] + sorted(
        os.path.join(csrc, f) for f in os.listdir(csrc) if f.endswith((".cuh", ".h")))
    return cu, hdr


def path(name: str) -> str:
    return os.path.join(OUT, f"libpolylla_{name}.so")


def _build_one(name, flags, cu, hdr, force):
    out = path(name)
    if not force and os.path.exists(out) and all(os.path.getmtime(s) <= os.path.getmtime(out) for s in cu + hdr):
        return out
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
           *flags, "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-I", os.path.join(ROOT, "include"),
           "-o", out, *cu]
    subprocess.run(cmd, check=True, cwd=ROOT, stdout=subprocess.DEVNULL)
    return out


def build_variants(names=None, force=False) -> dict:
    """Build (if stale) and return {name: path}."""
    os.makedirs(OUT, exist_ok=True)
    cu, hdr = _sources()
    names = list(VARIANTS) if names is None else list(names)
    with ThreadPoolExecutor(max_workers=len(names)) as ex:
        futs = {n: ex.submit(_build_one, n, VARIANTS[n], cu, hdr, force) for n in names}
        return {n: f.result() for n, f in futs.items()}
