# A/B of several variants (per-kernel medians, config $1): libpolylla.so vs libpolylla_$2.so ...
c=$1; shift
L=$PWD/paper_2403_14723_b200
args="$L/libpolylla.so"; for v in "$@"; do args="$args $L/libpolylla_$v.so"; done
timeout 900 python tools/kernel_times.py $c 30 $args $args 2>&1 | grep -v Warn | grep -v counts
