timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/bench_c3.json 2>gpurun_out/bench_c3.err; tail -2 gpurun_out/bench_c3.err
timeout 600 python bench.py --config 5 --steps 5 --warmup 2 > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err
timeout 900 python bench.py --config 4 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_c4.json 2>gpurun_out/bench_c4.err; tail -2 gpurun_out/bench_c4.err
for c in 3 5 4; do python -c "
import json,sys; d=json.load(open('gpurun_out/bench_c$c.json')); print('cfg$c ms/step %.3f  Gtris/s %.2f  pipe_frac %.3f e2e %s cpu %s' % (d['ms_per_step'], d['value']/1e9, d['pipeline_roofline']['frac'], d['e2e'] and round(d['e2e']['value']/1e9,3), d['cpu_baseline'] and round(d['cpu_baseline']['value']/1e6,3))); print({k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}); print(d['config']['per_mesh_rank0'], d['clocks'])"; done
