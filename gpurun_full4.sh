mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); print('ms/step %.3f  Gtris/s %.2f  pipe_frac %.3f' % (d['ms_per_step'], d['value']/1e9, d['pipeline_roofline']['frac'])); print({k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}); print(d['e2e'])"
