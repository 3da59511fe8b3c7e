# config 5 batch time vs the number of streams (lanes)
for n in 1 2 3 4 6; do POLYLLA_BENCH_LANES=$n timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-pcie 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('lanes', $n, round(d['ms_per_step'],2), d['config'].get('launch_mode', d.get('launch_mode')))"; done
