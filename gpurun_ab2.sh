mkdir -p gpurun_out
POLYLLA_LIB=$PWD/paper_2403_14723_b200/libpolylla_stage.so timeout 900 python -m pytest tests -m gpu -x -q -k "config3_full or config2 or fan or random or config5 or tie or square or grid or host" 2>&1 | tail -2
timeout 600 python tools/kernel_times.py 3 40 $PWD/paper_2403_14723_b200/libpolylla.so $PWD/paper_2403_14723_b200/libpolylla_stage.so 2>&1 | grep -v Warn
timeout 600 python tools/kernel_times.py 5 20 $PWD/paper_2403_14723_b200/libpolylla.so $PWD/paper_2403_14723_b200/libpolylla_stage.so 2>&1 | grep -v Warn
