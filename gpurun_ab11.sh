mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 $L/libpolylla.so $L/libpolylla_prev.so $L/libpolylla.so $L/libpolylla_prev.so 2>&1 | grep -v Warn
