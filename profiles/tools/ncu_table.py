"""Extract the headline metrics of an `ncu --set full` report (raw page CSV) per kernel.
usage: ncu -i X.ncu-rep --page raw --csv > raw.csv; python ncu_table.py raw.csv > table.csv"""
import csv
import sys

WANT = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__t_sector_hit_rate.pct',
        'l1tex__t_sector_hit_rate.pct', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'launch__registers_per_thread', 'launch__occupancy_limit_shared_mem',
        'smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio']

rows = list(csv.reader(open(sys.argv[1])))
hdr, units = rows[0], rows[1]
w = csv.writer(sys.stdout)
w.writerow(['kernel'] + WANT)
for r in rows[2:]:
    out = [r[hdr.index('Kernel Name')].split('(')[0]]
    for x in WANT:
        out.append((r[hdr.index(x)] + ' ' + units[hdr.index(x)]).strip() if x in hdr else 'n/a')
    w.writerow(out)
