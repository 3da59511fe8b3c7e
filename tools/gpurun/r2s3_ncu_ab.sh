# ncu headline metrics of k_tile: libpolylla.so vs libpolylla_$1.so (config 3, one launch each)
mkdir -p gpurun_out/ncu
L=$PWD/paper_2403_14723_b200
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__warps_active.avg.per_cycle_active,dram__bytes_read.sum,dram__bytes_write.sum
for lib in libpolylla.so libpolylla_$1.so; do
  POLYLLA_LIB=$L/$lib timeout 900 ncu --metrics $M --clock-control none -k regex:"^k_tile$" -c 1 --csv python tools/kernel_times.py 3 2 > gpurun_out/ncu/$lib.csv 2>/dev/null
  echo "== $lib"; grep -E '"(smsp|gpu|l1tex|dram)__' gpurun_out/ncu/$lib.csv | awk -F'","' '{print $(NF-2), $NF}' | tr -d '"'
done
