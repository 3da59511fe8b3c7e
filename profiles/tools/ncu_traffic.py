"""Write profiles/ncu_traffic.json: DRAM bytes (read + write) per launch of each kernel
group, from an ncu capture of THIS source tree (bench.py reports it as roofline.traffic
only while the source hash matches).

usage: python profiles/tools/ncu_traffic.py CONFIG capture.csv [capture.csv ...]
  capture.csv: `ncu --csv` output in the launch-list layout (one row per launch and metric,
  e.g. `--metrics dram__bytes_read.sum,dram__bytes_write.sum` or a `--set full` capture
  exported with `ncu -i X.ncu-rep --page raw --csv` is NOT this layout: use the launch list)."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from bench import src_hash  # noqa: E402

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
# kernel -> the bench/profile group it is timed in (polylla_profile_* marks)
GROUP = {"k_tile": "k_tile", "k_hash_clear": "k_left_match", "k_left_insert": "k_left_match",
         "k_border_rank": "k_left_match", "k_border_scan": "k_border_scan", "k_border_emit": "k_border_scan",
         "k_border_next": "k_border_next", "k_label_fixup": "k_label_fixup", "k_repair_mid": "k_repair",
         "k_repair_rewire": "k_repair", "k_seed_walk": "k_seed_walk", "k_canon_tiles": "k_canon_scan",
         "k_tiles_scan": "k_canon_scan", "k_emit": "k_extract"}


def main(cfg, paths):
    per_kernel = collections.defaultdict(list)  # kernel -> [bytes per launch]
    for path in paths:
        launches = collections.defaultdict(dict)
        for r in csv.reader(open(path)):
            if len(r) < 15 or r[0] == "ID":
                continue
            name = r[4].split("(")[0].replace("void ", "").replace("polylla::", "").split("<")[0]  # (k_tile<0>)
            if r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                launches[(r[0], name)][r[12]] = float(r[14].replace(",", "")) * SCALE.get(r[13], 1.0)
        for (lid, name), m in launches.items():
            if name in GROUP and len(m) == 2:
                per_kernel[name].append(m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"])
    groups = collections.defaultdict(float)
    for k, v in per_kernel.items():
        groups[GROUP[k]] += sum(v) / len(v)
    out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = {}
    if os.path.exists(out_path):
        d = json.load(open(out_path))
        if d.get("src_hash") != src_hash():
            d = {}
    d["src_hash"] = src_hash()
    d["source"] = ", ".join(os.path.relpath(p, ROOT) for p in paths) + \
        " (ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum; mean per launch, summed per group)"
    d[f"config{cfg}"] = {k: round(v) for k, v in sorted(groups.items())}
    json.dump(d, open(out_path, "w"), indent=1)
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main(int(sys.argv[1]), sys.argv[2:])
