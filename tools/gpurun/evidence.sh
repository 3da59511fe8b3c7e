set -x
mkdir -p gpurun_out/ev
nproc > gpurun_out/ev/host.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> gpurun_out/ev/host.txt; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv >> gpurun_out/ev/host.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.txt 2>&1; tail -2 gpurun_out/ev/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/ev/bench_c3.json 2> gpurun_out/ev/bench_c3.err
timeout 900 python bench.py --config 2 > gpurun_out/ev/bench_c2.json 2> gpurun_out/ev/bench_c2.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > gpurun_out/ev/bench_c5.json 2> gpurun_out/ev/bench_c5.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ev/bench_c4.json 2> gpurun_out/ev/bench_c4.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.err
timeout 600 python tools/kernel_times.py 3 40 > gpurun_out/ev/kernel_times_c3.txt 2>&1
timeout 300 python tools/regions_time.py > gpurun_out/ev/regions_time_c3.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$|^k_emit$|^k_seed_walk$|^k_label_fixup$" -c 4 -o gpurun_out/ev/prof_c3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ls -la gpurun_out/ev
