# A/B: fast GPU suite on libpolylla.so, then per-kernel medians of libpolylla.so vs libpolylla_$1.so on configs 3 and 5
mkdir -p gpurun_out/ab
L=$PWD/paper_2403_14723_b200
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/ab/pytest.txt 2>&1; tail -5 gpurun_out/ab/pytest.txt
for c in 3 5; do timeout 900 python tools/kernel_times.py $c 30 $L/libpolylla.so $L/libpolylla_$1.so $L/libpolylla.so $L/libpolylla_$1.so 2>&1 | grep -v Warn; done > gpurun_out/ab/kt.txt; cat gpurun_out/ab/kt.txt
