timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "triangle_polygons or call_order" 2>&1 | tail -2
timeout 300 python tools/regions_time.py 2>&1 | grep cfg3
bash tools/gpurun/sanitizer.sh
