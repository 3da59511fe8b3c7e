# session 4: fast GPU suite on libpolylla.so, then per-kernel medians vs variants on config $1
c=$1; shift
mkdir -p gpurun_out/ab
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/ab/pytest.txt 2>&1; tail -3 gpurun_out/ab/pytest.txt
bash tools/gpurun/r2s3_ab2.sh $c "$@" > gpurun_out/ab/kt_c$c.txt 2>&1; cat gpurun_out/ab/kt_c$c.txt
