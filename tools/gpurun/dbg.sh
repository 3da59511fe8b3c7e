timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "triangle_polygons" 2>&1 | tail -2
timeout 300 python tools/regions_time.py 2>&1 | grep cfg3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_uf -c 4 --csv python tools/regions_time.py 2>&1 | grep k_uf | awk -F'","' '{print $5, $(NF-2), $NF}' | head -20
