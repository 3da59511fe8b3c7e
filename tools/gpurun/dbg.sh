timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "triangle_polygons or call_order" 2>&1 | grep -v "^\s*$" | tail -15
