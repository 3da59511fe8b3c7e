# per-kernel medians on config 3 for libpolylla.so and each variant named in $@
L=$PWD/paper_2403_14723_b200
libs="$L/libpolylla.so"; for v in "$@"; do libs="$libs $L/libpolylla_$v.so"; done
timeout 1200 python tools/kernel_times.py 3 30 $libs $libs 2>&1 | grep -v Warn | grep -v counts
