# configs 4 and 5 bench lines (kernel-only) + per-kernel medians of config 5
mkdir -p gpurun_out/c45
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c45/bench_c5.json 2> gpurun_out/c45/bench_c5.err; tail -c 300 gpurun_out/c45/bench_c5.err
timeout 1200 python bench.py --config 4 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c45/bench_c4.json 2> gpurun_out/c45/bench_c4.err; tail -c 300 gpurun_out/c45/bench_c4.err
for f in gpurun_out/c45/bench_c*.json; do python -c "import json; d=json.load(open('$f')); print('$f', d['ms_per_step'], d['roofline']['kernel'], round(d['roofline']['frac'],4), d.get('kernels_ms_per_step'))"; done
