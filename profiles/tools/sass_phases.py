"""Per-phase aggregation of an `ncu --page source --csv` SASS dump: the kernel body is
cut at its BAR.SYNC instructions (phase boundaries of k_tile); for each segment print
warp instructions executed, stall samples and the top stall reasons.
usage: python sass_phases.py source.csv"""
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ix = {k: i for i, k in enumerate(hdr)}
    stalls = [k for k in hdr if k.startswith("stall_")]
    segs, cur = [], {"start": None, "inst": 0, "samp": 0, "st": {k: 0 for k in stalls}, "n": 0}
    tot_inst = tot_samp = 0
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        if cur["start"] is None:
            cur["start"] = r[ix["Address"]]
        inst = int(r[ix["Instructions Executed"]] or 0)
        samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        cur["inst"] += inst
        cur["samp"] += samp
        cur["n"] += 1
        tot_inst += inst
        tot_samp += samp
        for k in stalls:
            cur["st"][k] += int(r[ix[k]] or 0)
        if src.startswith("BAR.SYNC") or src.startswith("EXIT") or src.startswith("RET"):
            cur["end"] = src.split()[0]
            segs.append(cur)
            cur = {"start": None, "inst": 0, "samp": 0, "st": {k: 0 for k in stalls}, "n": 0}
    for i, s in enumerate(segs):
        if s["inst"] == 0 and s["samp"] == 0:
            continue
        top = sorted(s["st"].items(), key=lambda kv: -kv[1])[:4]
        print(f"seg{i:2d} n={s['n']:4d} inst {100 * s['inst'] / tot_inst:5.1f}%  samples {100 * s['samp'] / tot_samp:5.1f}%  "
              + " ".join(f"{k[6:]}={100 * v / max(1, s['samp']):.0f}%" for k, v in top) + f"  [{s['end']}]")
    agg = {k: sum(s["st"][k] for s in segs) for k in stalls}
    print("total: " + " ".join(f"{k[6:]}={100 * v / tot_samp:.1f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:10]))


if __name__ == "__main__":
    main(sys.argv[1])
