# round 2: fast GPU suite (no slow tests) + per-kernel medians on config 3
mkdir -p gpurun_out/q
(free -g; nproc; lscpu | grep -E "Model name|^CPU\(s\)"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/q/host.txt 2>&1
timeout 1500 python -m pytest tests -m "gpu and not slow" -q -x -p no:cacheprovider > gpurun_out/q/pytest.txt 2>&1; tail -3 gpurun_out/q/pytest.txt
timeout 600 python tools/kernel_times.py 3 30 > gpurun_out/q/kt.txt 2>&1; cat gpurun_out/q/kt.txt | grep -v Warn
