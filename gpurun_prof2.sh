mkdir -p gpurun_out/p2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$|^k_emit$|^k_seed_walk$|^k_repair_mid$|^k_repair_rewire$|^k_left_insert$" -c 6 -o gpurun_out/p2/prof python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > gpurun_out/p2/ncu.log 2>&1
tail -3 gpurun_out/p2/ncu.log
