# round 2: fast GPU suite + A/B per-kernel medians of libpolylla.so vs a variant ($1)
mkdir -p gpurun_out/ab
L=$PWD/paper_2403_14723_b200
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/ab/pytest.txt 2>&1; tail -3 gpurun_out/ab/pytest.txt
timeout 900 python tools/kernel_times.py 3 30 $L/libpolylla.so $L/libpolylla_$1.so $L/libpolylla.so $L/libpolylla_$1.so > gpurun_out/ab/kt.txt 2>&1; grep -v Warn gpurun_out/ab/kt.txt
