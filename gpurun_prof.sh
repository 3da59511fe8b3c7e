mkdir -p gpurun_out
timeout 300 python tools/phase_timing.py 3 > gpurun_out/phase_c3.txt 2>&1; tail -12 gpurun_out/phase_c3.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -c 1 -o gpurun_out/prof_tile python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ls -la gpurun_out
