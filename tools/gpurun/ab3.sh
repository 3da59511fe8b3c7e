mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 600 python tools/kernel_times.py 3 30 $L/libpolylla.so $L/libpolylla_f384.so $L/libpolylla_f512.so $L/libpolylla_f128.so 2>&1 | grep -v Warn
timeout 600 python tools/kernel_times.py 5 15 $L/libpolylla.so $L/libpolylla_f384.so $L/libpolylla_f512.so $L/libpolylla_f128.so 2>&1 | grep -v Warn
