timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 10 python tools/sanitize_run.py > gpurun_out/san_racecheck.txt 2>&1; echo "racecheck rc=$?"; tail -3 gpurun_out/san_racecheck.txt
bash gpurun_quick5.sh
