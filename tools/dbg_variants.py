"""Debug: run the schedule-test meshes through each given library (path list), report the
first failing mesh per library."""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from test_gpu_schedule import _meshes  # noqa: E402
from test_gpu_parity import assert_parity  # noqa: E402
from paper_2403_14723_b200 import polylla as pp  # noqa: E402

for lib in sys.argv[1:]:
    pp.set_library(lib)
    for name, (xy, tri) in _meshes().items():
        try:
            assert_parity(xy, tri, invariants=False)
        except Exception as e:  # noqa: BLE001
            print(os.path.basename(lib), name, "FAIL", repr(e)[:300], flush=True)
            try:
                import torch
                torch.cuda.synchronize()
                print("sync ok")
            except Exception as e2:  # noqa: BLE001
                print("sync:", repr(e2)[:200])
            break
    else:
        print(os.path.basename(lib), "ok", flush=True)
