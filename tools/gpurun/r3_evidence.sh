# round 2 session 4 evidence (profiles/r02s4): host, full GPU suite, smoke, ncu launch list -> ncu_traffic.json
# (this source hash), bench lines (c3 default, c2, c2 shuffled, c5, c4, reference arm),
# per-kernel medians, ncu --set full of the top kernels
O=gpurun_out/ev5; mkdir -p $O
(nproc; lscpu | grep -E "Model name|^CPU\(s\)"; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > $O/host.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c3.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
python profiles/tools/summarize_launches.py $O/launches_c3.csv --only-prefix polylla:: > $O/launches_c3_summary.txt 2>&1; head -20 $O/launches_c3_summary.txt
python profiles/tools/ncu_traffic.py 3 $O/launches_c3.csv > $O/ncu_traffic.txt 2>&1; cp profiles/ncu_traffic.json $O/
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --config 2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 900 python bench.py --config 2 --order shuffled --no-cpu-baseline > $O/bench_c2_shuffled.json 2> $O/bench_c2_shuffled.err
timeout 900 python bench.py --config 2 --order shuffled --sort --no-cpu-baseline --no-e2e > $O/bench_c2_shuffled_sort.json 2> $O/bench_c2_shuffled_sort.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > $O/bench_c4.json 2> $O/bench_c4.err
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-row-hint > $O/bench_c5_contiguous.json 2> $O/bench_c5_contiguous.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-row-hint > $O/bench_c4_contiguous.json 2> $O/bench_c4_contiguous.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
(for c in 3 5; do timeout 600 python tools/kernel_times.py $c 40 2>&1 | grep -v Warn; done; POLYLLA_ROWS=1 timeout 600 python tools/kernel_times.py 5 40 2>&1 | grep -v Warn) > $O/kernel_times.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$|^k_emit$|^k_seed_walk$|^k_label_fixup$" -c 4 -o $O/prof_c3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
ncu -i $O/prof_c3.ncu-rep --page raw --csv > $O/prof_c3_raw.csv 2>&1; python profiles/tools/ncu_table.py $O/prof_c3_raw.csv > $O/ncu_full_c3.csv 2>&1; rm -f $O/prof_c3_raw.csv
for f in $O/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', d.get('impl','ours'), round(d['ms_per_step'],3), d.get('roofline',{}).get('kernel'), d.get('roofline',{}).get('frac'), d.get('roofline',{}).get('traffic'))" 2>&1 | tail -1; done
ls -la $O
