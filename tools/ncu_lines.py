"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an ncu report
(ncu --page source --print-source cuda,sass).  usage: python tools/ncu_lines.py REPORT KERNEL_REGEX [N]"""
import csv, subprocess, sys
rep, kre = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", "regex:" + kre, "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, rows, hdr = None, [], None
for x in csv.reader(out.splitlines()):
    if len(x) == 2 and x[0] == "File Path":
        fname = x[1].split("/")[-1]
    elif x and x[0] == "Line No":
        hdr = x
    elif hdr and len(x) == len(hdr) and x[0] not in ("", "-"):
        rows.append((fname, x))
iI = hdr.index("Instructions Executed"); iS = hdr.index("Warp Stall Sampling (All Samples)")
num = lambda v: float(v) if v not in ("", "-") else 0.0
totI = sum(num(x[iI]) for _, x in rows); totS = sum(num(x[iS]) for _, x in rows)
print(f"total warp instructions {totI:.0f}, samples {totS:.0f}")
for f, x in sorted(rows, key=lambda r: -num(r[1][iI]))[:N]:
    print(f"{100*num(x[iI])/totI:5.1f}% inst {100*num(x[iS])/max(totS,1):5.1f}% stall  {f}:{x[0]:>4}  {x[1].strip()[:90]}")
