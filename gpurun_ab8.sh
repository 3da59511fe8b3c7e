mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 900 python -m pytest tests -m gpu -x -q -k "config3_full or config2 or fan or random or config5 or tie or square or grid or host" 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 $L/libpolylla.so $L/libpolylla_prev.so $L/libpolylla.so $L/libpolylla_prev.so 2>&1 | grep -v Warn
