mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 2>&1 | grep -v Warn
timeout 600 python tools/kernel_times.py 5 20 2>&1 | grep -v Warn
