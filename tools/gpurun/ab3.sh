mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 600 python tools/kernel_times.py 3 30 $L/libpolylla.so $L/libpolylla_s128.so $L/libpolylla_s512.so $L/libpolylla_s384.so 2>&1 | grep -v Warn
