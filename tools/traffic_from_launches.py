"""Per-layer DRAM traffic and time of the pipe kernel(s) from an ncu launch list
(tools/profile_round.sh): median per kernel variant (split layers: the A-only and
B-only launches, told apart by the MODE template argument), summed over one layer.

usage: python tools/traffic_from_launches.py CONFIG launches.csv [profiles/roofline_traffic.json]
"""
import csv
import json
import statistics
import sys
from collections import defaultdict


def main():
    cfg, path = sys.argv[1], sys.argv[2]
    out = sys.argv[3] if len(sys.argv) > 3 else None
    rows = [ln for ln in open(path) if ln.startswith('"')]
    per = defaultdict(lambda: defaultdict(dict))  # kernel -> launch id -> metric -> value
    for r in csv.DictReader(rows):
        if "pipe_" not in r["Kernel Name"]:
            continue
        per[r["Kernel Name"]][r["ID"]][r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    res = {"kernels": {}}
    tot = defaultdict(float)
    for name, launches in per.items():
        med = {m: statistics.median(v[m] for v in launches.values()) for m in next(iter(launches.values()))}
        short = name.split("(")[0].replace("void ", "")
        res["kernels"][short] = {"launches": len(launches), **{k: int(v) for k, v in med.items()}}
        for k, v in med.items():
            tot[k] += v
    res["dram_read"] = int(tot["dram__bytes_read.sum"])
    res["dram_write"] = int(tot["dram__bytes_write.sum"])
    res["dram_bytes_per_launch"] = res["dram_read"] + res["dram_write"]
    res["ncu_time_ns_per_layer"] = int(tot["gpu__time_duration.sum"])
    print(json.dumps({cfg: res}, indent=1))
    if out:
        try:
            cur = json.load(open(out))
        except (OSError, ValueError):
            cur = {}
        old = cur.get(cfg, {})
        if "algorithmic_bytes_per_launch" in old:
            res["algorithmic_bytes_per_launch"] = old["algorithmic_bytes_per_launch"]
        cur[cfg] = res
        json.dump(cur, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
