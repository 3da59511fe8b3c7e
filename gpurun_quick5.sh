timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in 3 5; do
timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps $([ $c = 5 ] && echo 3 || echo 100) --warmup 2 > gpurun_out/bench_q$c.json 2>gpurun_out/bench_q$c.err; tail -2 gpurun_out/bench_q$c.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q$c.json')); print('cfg$c ms/step %.3f  Gtris/s %.2f  pipe_frac %.3f' % (d['ms_per_step'], d['value']/1e9, d['pipeline_roofline']['frac'])); print({k: round(v,3) for k,v in d['kernels_ms_per_step'].items()})"
done
