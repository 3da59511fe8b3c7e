# non-slow GPU suite, bench config 3, ncu --set full of k_tile (source + warp state), launch list
mkdir -p gpurun_out/prof
timeout 1200 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/prof/pytest.txt 2>&1; tail -3 gpurun_out/prof/pytest.txt
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/prof/bench_c3.json 2> gpurun_out/prof/bench_c3.err; tail -c 600 gpurun_out/prof/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$" -c 1 -o gpurun_out/prof/tile python tools/kernel_times.py 3 2 > /dev/null 2>&1
ncu -i gpurun_out/prof/tile.ncu-rep --page details --csv > gpurun_out/prof/tile_details.csv 2>&1
ncu -i gpurun_out/prof/tile.ncu-rep --page source --csv > gpurun_out/prof/tile_source.csv 2>&1
ls -la gpurun_out/prof
