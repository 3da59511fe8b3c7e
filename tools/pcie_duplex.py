"""PCIe check for the end-to-end pipeline: pinned H2D and D2H alone and concurrently (two
streams), with the per-mesh byte counts of config 3 (400 MB up, 838 MB down)."""
import time

import torch

up_b, down_b = 399_848_356, 838_315_796
h_up = torch.empty(up_b, dtype=torch.uint8).pin_memory()
h_down = torch.empty(down_b, dtype=torch.uint8).pin_memory()
d_up = torch.empty(up_b, dtype=torch.uint8, device="cuda")
d_down = torch.empty(down_b, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def up():
    with torch.cuda.stream(s1):
        d_up.copy_(h_up, non_blocking=True)


def down():
    with torch.cuda.stream(s2):
        h_down.copy_(d_down, non_blocking=True)


def both():
    up()
    down()


tu, td, tb = timed(up), timed(down), timed(both)
print(f"H2D {up_b / 1e6:.0f} MB: {tu:.2f} ms ({up_b / tu / 1e6:.1f} GB/s)")
print(f"D2H {down_b / 1e6:.0f} MB: {td:.2f} ms ({down_b / td / 1e6:.1f} GB/s)")
print(f"both concurrently: {tb:.2f} ms (ideal max = {max(tu, td):.2f} ms; aggregate {(up_b + down_b) / tb / 1e6:.1f} GB/s)")
