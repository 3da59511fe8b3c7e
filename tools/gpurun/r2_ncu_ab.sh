# ncu metrics of k_tile (and the rest) for libpolylla.so vs a variant ($1), config 3
mkdir -p gpurun_out/ncuab
L=$PWD/paper_2403_14723_b200
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum
for lib in libpolylla.so libpolylla_$1.so; do
  timeout 600 ncu --metrics $M --clock-control none --csv -k regex:"k_tile|k_xy32" -c 4 --log-file gpurun_out/ncuab/$lib.csv python tools/kernel_times.py 3 2 $L/$lib > gpurun_out/ncuab/$lib.log 2>&1
done
python profiles/tools/summarize_launches.py gpurun_out/ncuab/libpolylla.so.csv 2>/dev/null | head -5
grep -v Warn gpurun_out/ncuab/*.log | grep counts
