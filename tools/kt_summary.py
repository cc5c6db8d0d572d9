"""Summarise tools/kt_ncu.sh CSVs: mean duration (us), warp instructions and warps active per kernel."""
import collections
import csv
import sys

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
    acc = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows[1:]:
        try:
            acc[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",", "")))
        except ValueError:
            pass
    print(path)
    tot = 0.0
    for k, m in sorted(acc.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        d = m["gpu__time_duration.sum"]
        mean = sum(d) / len(d)
        tot += mean
        ins = m.get("smsp__inst_executed.sum", [0])
        wa = m.get("sm__warps_active.avg.pct_of_peak_sustained_active", [0])
        print(f"  {k[:60]:60s} n={len(d):3d} {mean:9.1f} us  {sum(ins)/len(ins)/1e6:8.2f}M inst  {sum(wa)/len(wa):5.1f}% warps")
    print(f"  total per iteration {tot:.1f} us")
