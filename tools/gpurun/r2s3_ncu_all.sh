# SURVEY 8(d) ncu rows: every kernel of one step on configs 2 and 3 (--set full, headline metrics)
O=gpurun_out/ncuall; mkdir -p $O
for c in 3 2; do
  timeout 1500 ncu --set full --clock-control none -k regex:"^k_" -c 20 -o $O/full_c$c python bench.py --config $c --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-graph --no-pcie > /dev/null 2>&1
  ncu -i $O/full_c$c.ncu-rep --page raw --csv > $O/raw_c$c.csv 2>&1
  python profiles/tools/ncu_table.py $O/raw_c$c.csv > $O/ncu_full_all_c$c.csv 2>&1; rm -f $O/raw_c$c.csv $O/full_c$c.ncu-rep
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-graph --no-pcie > /dev/null 2>&1
  python profiles/tools/summarize_launches.py $O/launches_c$c.csv --only-prefix polylla:: > $O/launches_c${c}_summary.txt 2>&1
done
wc -l $O/*.csv; head -30 $O/ncu_full_all_c3.csv | cut -c1-200
