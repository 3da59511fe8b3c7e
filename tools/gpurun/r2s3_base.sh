# round 2 session 3: baseline of the restored tree: fast GPU suite, per-kernel medians c3/c5, bench c3
mkdir -p gpurun_out/base
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/base/pytest.txt 2>&1; tail -3 gpurun_out/base/pytest.txt
for c in 3 5; do timeout 600 python tools/kernel_times.py $c 30 2>&1 | grep -v Warn; done > gpurun_out/base/kt.txt; cat gpurun_out/base/kt.txt
timeout 900 python bench.py --steps 50 --warmup 5 > gpurun_out/base/bench_c3.json 2> gpurun_out/base/bench_c3.err; tail -c 300 gpurun_out/base/bench_c3.err
