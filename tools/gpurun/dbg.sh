timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config3_triangle_polygons" 2>&1 | grep -v "^\s*$" | tail -8
