mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | grep -v "^\s*$" | tail -15
timeout 300 python tools/regions_time.py 2>&1 | tail -2
bash tools/gpurun/sanitizer.sh
tail -n 3 gpurun_out/san/*.txt
