mkdir -p gpurun_out/p3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$" -c 1 -o gpurun_out/p3/prof python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/p3/ncu.log 2>&1
tail -2 gpurun_out/p3/ncu.log
