mkdir -p gpurun_out
L=$PWD/paper_2403_14723_b200
timeout 900 python tools/kernel_times.py 3 20 $L/libpolylla.so $L/libpolylla_koGATHER.so $L/libpolylla_koPF.so $L/libpolylla_koP4A.so $L/libpolylla_koP6.so 2>&1 | grep -v Warn
