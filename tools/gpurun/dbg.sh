L=$PWD/paper_2403_14723_b200
for v in libpolylla libpolylla_uf256 libpolylla_uf384 libpolylla_uf1024 libpolylla; do
  echo -n "$v: "; POLYLLA_LIB=$L/$v.so timeout 300 python tools/regions_time.py 2>&1 | grep cfg3
done
POLYLLA_LIB=$L/libpolylla_uf256.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "triangle_polygons and not config3" 2>&1 | tail -1
