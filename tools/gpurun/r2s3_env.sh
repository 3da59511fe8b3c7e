# env A/B: per-kernel medians of libpolylla.so on config $1 under VAR=value settings ($2 = VAR, rest = values)
mkdir -p gpurun_out/env
c=$1; var=$2; shift 2
for v in "$@"; do echo "== $var=$v"; env $var=$v timeout 600 python tools/kernel_times.py $c 30 2>&1 | grep -v Warn | grep -v counts; done > gpurun_out/env/kt_$var.txt; cat gpurun_out/env/kt_$var.txt
