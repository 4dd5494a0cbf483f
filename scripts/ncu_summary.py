"""Summarise an ncu --set full report: key metrics + SASS opcode mix."""
import csv
import subprocess
import sys
from collections import Counter

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "smsp__inst_executed.sum", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals)}


def opmix(rep, top=14):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    c = Counter()
    for r in rows[2:]:
        if not r[ia].isdigit():
            continue
        t = r[isrc].split()
        op = (t[1] if t and t[0].startswith("@") else (t[0] if t else "")).split(".")[0]
        c[op] += int(r[ia])
    tot = sum(c.values())
    return tot, c.most_common(top)


if __name__ == "__main__":
    for rep in sys.argv[1:]:
        m = raw(rep)
        print(f"== {rep}  kernel={m.get('Kernel Name', ('?',))[0][:90]}")
        for k in KEYS:
            if k in m:
                print(f"  {k:75s} {m[k][0]:>16s} {m[k][1]}")
        tot, mix = opmix(rep)
        print(f"  warp instructions: {tot}")
        print("  " + ", ".join(f"{k}:{v}" for k, v in mix))
