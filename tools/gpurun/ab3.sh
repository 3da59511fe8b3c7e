mkdir -p gpurun_out
for c in -1 0 10 25 50 100; do
POLYLLA_EMIT_CARVEOUT=$c timeout 600 python tools/kernel_times.py 3 30 2>&1 | grep -v Warn | sed "s/^/carve $c: /"
done
