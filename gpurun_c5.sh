mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "concurrent or config5" 2>&1 | tail -2
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err; tail -2 gpurun_out/bench_c5b.err
python -c "
import json; d=json.load(open('gpurun_out/bench_c5b.json')); print('c5 ms/step %.3f  Gtris/s %.2f  pipe_frac %.3f' % (d['ms_per_step'], d['value']/1e9, d['pipeline_roofline']['frac']), d['launch_mode'])"
