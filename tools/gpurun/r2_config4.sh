# config 4 bit-exact against the oracle (~100 GB host RAM), plus the slow GPU tests
mkdir -p gpurun_out/c4
(free -g; nproc; lscpu | grep -E "Model name") > gpurun_out/c4/host.txt 2>&1
POLYLLA_HUGE=1 timeout 3600 python -m pytest tests/test_gpu_config4.py -s -q -p no:cacheprovider > gpurun_out/c4/config4_oracle.txt 2>&1; tail -5 gpurun_out/c4/config4_oracle.txt
timeout 1800 python -m pytest tests -m "gpu and slow" -q -p no:cacheprovider > gpurun_out/c4/pytest_slow.txt 2>&1; tail -3 gpurun_out/c4/pytest_slow.txt
