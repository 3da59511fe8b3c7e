# compute-sanitizer over tests/sanitize_run.py (small meshes, every case checked against the oracle)
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $t --error-exitcode 9 --print-limit 200 python tests/sanitize_run.py > gpurun_out/san/san_$t.txt 2>&1
  echo "$t rc=$?"; tail -2 gpurun_out/san/san_$t.txt
done
