# session 4: the full GPU suite (slow tests included) + sanitizer + smoke
mkdir -p gpurun_out/full
timeout 3000 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/full/pytest_gpu.txt 2>&1; tail -3 gpurun_out/full/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full/smoke.txt 2>&1; echo smoke rc=$?
bash tools/gpurun/sanitizer.sh
