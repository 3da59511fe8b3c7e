set -x
nproc > gpurun_out/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/host.txt; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv >> gpurun_out/host.txt
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config 2 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile|k_label_fixup|k_extract|k_seed_walk" -c 4 -o gpurun_out/prof_c3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
ls -la gpurun_out
