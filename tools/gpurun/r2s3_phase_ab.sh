# per-phase k_tile clocks: current tree vs the tree in oldsrc_ab/ (config 3)
mkdir -p gpurun_out/ph
timeout 600 python tools/phase_timing.py 3 > gpurun_out/ph/new.txt 2>&1; tail -9 gpurun_out/ph/new.txt
POLYLLA_SRC=$PWD/oldsrc_ab timeout 600 python tools/phase_timing.py 3 > gpurun_out/ph/old.txt 2>&1; tail -9 gpurun_out/ph/old.txt
