"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel
name: launches, total us, mean us.  Used to compare the TTFT forward's
kernel mix between the bf16 and MX paths (profiles/r02/ttft_breakdown).

    python scripts/kernel_breakdown.py launches.csv [--per N]
"""
import collections
import csv
import json
import sys


def main():
    path = sys.argv[1]
    per = int(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))
            if r.get("Metric Name") == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        name = r["Kernel Name"]
        name = name.split("(")[0][:90]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else v
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(v[1] for v in agg.values())
    for name, (cnt, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(json.dumps({"kernel": name, "launches": cnt // per, "us": round(us / per, 1),
                          "mean_us": round(us / cnt, 2), "share": round(us / tot, 4)}))
    print(json.dumps({"total_us": round(tot / per, 1), "launches": len(rows) // per}))


if __name__ == "__main__":
    main()
