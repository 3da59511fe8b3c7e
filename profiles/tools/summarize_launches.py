"""Summarise an ncu launch list (gpu__time_duration per launch) into per-kernel shares.
usage: python tools_summarize.py launches.csv [steps_to_skip]"""
import collections
import csv
import sys


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    per = collections.OrderedDict()
    for r in rows:
        name = r[4].split("(")[0].split("<")[0]
        if "k_scan" in r[4]:
            name = r[4].split("(")[0]
        per.setdefault(name, []).append(float(r[-1]) / 1e3)
    tot = sum(sum(v) for v in per.values())
    print(f"{'kernel':45s} {'launches':>8s} {'avg us':>10s} {'share':>7s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        print(f"{k:45s} {len(v):8d} {sum(v)/len(v):10.1f} {100*sum(v)/tot:6.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
