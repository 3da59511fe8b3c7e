"""Per-CUDA-source-line stall samples and executed instructions from an ncu report.
usage: ncu -i X.ncu-rep --page source --csv --print-source cuda,sass -k K > cs.csv
       python ncu_lines.py cs.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
hdr = rows[hdr_i]
S = hdr.index("Warp Stall Sampling (All Samples)")
I = hdr.index("Instructions Executed")
src = {}
samp = collections.Counter()
inst = collections.Counter()
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr) or not r[0].isdigit():
        continue  # SASS rows follow their source line; the line row carries the totals
    ln = int(r[0])
    src[ln] = r[1]
    samp[ln] += int(r[S]) if r[S].isdigit() else 0
    inst[ln] += int(r[I]) if r[I].isdigit() else 0
tot = sum(samp.values())
tinst = sum(inst.values())
print(f"total samples {tot}, warp instructions {tinst}")
for ln, s in samp.most_common(top):
    print(f"{s:7d} {100*s/tot:5.1f}%  inst {100*inst[ln]/max(tinst,1):5.1f}%  L{ln:<4d} {src.get(ln,'').strip()[:90]}")
