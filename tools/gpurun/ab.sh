mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 $L/libpolylla.so $L/libpolylla_prev.so $L/libpolylla.so $L/libpolylla_prev.so 2>&1 | grep -v Warn
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['ms_per_step'], d['config']['per_mesh_rank0'])"
