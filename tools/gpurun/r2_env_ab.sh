# A/B of one library under two environment settings: $1="VAR=a" $2="VAR=b" (config 3 medians + ncu k_tile metrics)
mkdir -p gpurun_out/envab
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for e in "$1" "$2" "$1" "$2"; do env $e timeout 600 python tools/kernel_times.py 3 30 2>&1 | grep -v Warn | sed "s/^/[$e] /"; done
for e in "$1" "$2"; do env $e timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"^k_tile$" -c 2 --log-file gpurun_out/envab/"$e".csv python tools/kernel_times.py 3 2 > /dev/null 2>&1; done
ls gpurun_out/envab
