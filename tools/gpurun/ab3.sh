mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 600 python tools/kernel_times.py 3 40 $L/libpolylla.so $L/libpolylla_p6f.so $L/libpolylla.so $L/libpolylla_p6f.so 2>&1 | grep -v Warn
