"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --csv`, one row per (launch, metric)) into per-kernel shares.
usage: python summarize_launches.py launches.csv [--only-prefix polylla::]"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main(path, prefix=""):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    launches = collections.OrderedDict()  # id -> {name, metrics}
    for r in rows:
        lid, kname, metric, unit, val = r[0], r[4], r[12], r[13], r[14]
        name = kname.split("(")[0]
        if name.startswith("void "):
            name = name[5:]
        d = launches.setdefault(lid, {"name": name, "m": {}})
        d["m"][metric] = float(val.replace(",", "")) * SCALE.get(unit, 1.0)
    per = collections.OrderedDict()
    for d in launches.values():
        if prefix and not d["name"].startswith(prefix):
            continue
        per.setdefault(d["name"], []).append(d["m"])
    tot = sum(sum(m.get("gpu__time_duration.sum", 0.0) for m in v) for v in per.values())
    print(f"{'kernel':42s} {'launches':>8s} {'us/launch':>10s} {'share':>7s} {'DRAM MB/launch':>15s} {'DRAM GB/s':>10s}")
    for k, v in sorted(per.items(), key=lambda kv: -sum(m.get("gpu__time_duration.sum", 0) for m in kv[1])):
        t = sum(m.get("gpu__time_duration.sum", 0.0) for m in v)
        b = sum(m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0) for m in v)
        print(f"{k:42s} {len(v):8d} {t / len(v):10.1f} {100 * t / tot:6.1f}% {b / len(v) / 1e6:15.1f} "
              f"{(b / (t * 1e-6) / 1e9) if t else 0:10.0f}")


if __name__ == "__main__":
    pre = sys.argv[sys.argv.index("--only-prefix") + 1] if "--only-prefix" in sys.argv else ""
    main(sys.argv[1], pre)
