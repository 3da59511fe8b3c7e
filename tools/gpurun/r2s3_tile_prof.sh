# k_tile diagnostics: per-phase clocks and the SASS per-phase instruction/stall split
mkdir -p gpurun_out/tp
timeout 600 python tools/phase_timing.py 3 > gpurun_out/tp/phase_c3.txt 2>&1; cat gpurun_out/tp/phase_c3.txt | tail -10
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_tile$" -c 1 -o gpurun_out/tp/tile python tools/kernel_times.py 3 2 > /dev/null 2>&1
ncu -i gpurun_out/tp/tile.ncu-rep --page source --csv --print-source sass > gpurun_out/tp/tile_sass.csv 2>&1
ncu -i gpurun_out/tp/tile.ncu-rep --page raw --csv > gpurun_out/tp/tile_raw.csv 2>&1
python profiles/tools/sass_phases.py gpurun_out/tp/tile_sass.csv > gpurun_out/tp/phases_sass.txt 2>&1; cat gpurun_out/tp/phases_sass.txt | head -40
