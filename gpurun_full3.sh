mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 100 > gpurun_out/bench_q.json 2>gpurun_out/bench_q.err; tail -2 gpurun_out/bench_q.err
python -c "
import json; d=json.load(open('gpurun_out/bench_q.json')); print('ms/step %.3f  Gtris/s %.2f  pipe_frac %.3f' % (d['ms_per_step'], d['value']/1e9, d['pipeline_roofline']['frac'])); print({k: round(v,3) for k,v in d['kernels_ms_per_step'].items()}); print(d['config']['per_mesh_rank0'])"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tile" -c 1 -o gpurun_out/prof_tile3 python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph > /dev/null 2>&1
