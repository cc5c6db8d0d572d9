"""Top stall-sampled SASS lines of one kernel in an ncu report (reads `ncu --page source`).
usage: python tools/ncu_hot.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = [x for x in r[2:] if len(x) == len(h)]
iS = h.index("Warp Stall Sampling (All Samples)"); iA = h.index("Address"); iSrc = h.index("Source")
val = lambda x: int(x[iS]) if x[iS].strip().isdigit() else 0
tot = sum(val(x) for x in rows)
print("total samples", tot, "instructions", len(rows))
for i, x in enumerate(rows):
    x.append(i)
for x in sorted(rows, key=lambda x: -val(x))[:N]:
    print(f"{val(x):6d} {100*val(x)/tot:5.1f}% #{x[-1]:5d} {x[iSrc][:100]}")
