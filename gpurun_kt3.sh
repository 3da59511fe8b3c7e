mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "config3_full or config2 or fan or random or config5 or tie or square or grid or repair" 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 2>&1 | grep -v Warn
timeout 600 python tools/kernel_times.py 5 20 2>&1 | grep -v Warn
