# GPU suite (not slow), NEXT-2 ablation timing, run_host single-call latency, config-2 sensitivity rows
mkdir -p gpurun_out/b
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/b/pytest.txt 2>&1; tail -3 gpurun_out/b/pytest.txt
for c in 3 5; do timeout 600 python tools/kernel_times.py $c 20 2>&1 | grep -v Warn | sed "s/^/[ours] /"; POLYLLA_PAPER=1 timeout 600 python tools/kernel_times.py $c 20 2>&1 | grep -v Warn | sed "s/^/[paper] /"; done
timeout 900 python bench.py --config 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b/bench_c2.json 2> gpurun_out/b/bench_c2.err
timeout 900 python bench.py --config 2 --order shuffled --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b/bench_c2_shuffled.json 2> gpurun_out/b/bench_c2_shuffled.err
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/b/bench_c3.json 2> gpurun_out/b/bench_c3.err
for f in gpurun_out/b/bench_*.json; do python -c "import json,sys; d=json.load(open('$f')); print('$f', round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],4), d['e2e'] and round(d['e2e']['ms_per_step'],2), d['e2e'] and round(d['e2e'].get('single_call_ms',0),2))"; done
