# A/B per-kernel medians of libpolylla.so vs libpolylla_$1.so on configs 3, 5 (one jittered 2000-grid) and 4
L=$PWD/paper_2403_14723_b200
for c in 3 5; do timeout 900 python tools/kernel_times.py $c 20 $L/libpolylla.so $L/libpolylla_$1.so $L/libpolylla.so $L/libpolylla_$1.so 2>&1 | grep -v Warn; done
timeout 900 python tools/kernel_times.py 4 5 $L/libpolylla.so $L/libpolylla_$1.so 2>&1 | grep -v Warn
