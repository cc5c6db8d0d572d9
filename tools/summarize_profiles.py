"""Summarise a gpurun ncu launch list (+ optional --set full reports) into profiles/<tag>.md."""
import collections, csv, subprocess, sys, os

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, agg = None, collections.defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d["Metric Name"] == "gpu__time_duration.sum":
                agg[d["Kernel Name"].split("(")[0]].append(float(d["Metric Value"]))
    return agg

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "lts__t_sector_hit_rate.pct"]

def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        res.append({w: (r[h.index(w)], units[h.index(w)]) for w in WANT if w in h} | {"name": r[h.index("Kernel Name")]})
    return res

args = sys.argv[1:]
traffic_out, fpl = None, 1
if "--traffic-json" in args:  # --traffic-json OUT FRAMES_PER_LAUNCH: per-frame DRAM bytes per phase for bench.py
    i = args.index("--traffic-json")
    traffic_out, fpl = args[i + 1], int(args[i + 2])
    del args[i:i + 3]
tag, launch_csv = args[0], args[1]
reps = args[2:]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
PHASE = {"k_sat1": "integral_images", "k_sat2": "integral_images", "k_sat3": "integral_images",
         "k_sat1w": "integral_images", "k_sat2p": "integral_images", "k_sat3w": "integral_images",
         "k_sat3x": "integral_images", "k_sat1x": "integral_images", "k_advect_uniq64": "region", "k_advect_uniq64s": "region",
         "k_region": "region", "k_row": "row"}
lines = [f"# ncu summary {tag}", "", "## Launch list (gpu__time_duration.sum, --clock-control none, serialised)", "",
         "| kernel | launches | mean (us) | share |", "|---|---|---|---|"]
agg = launches(launch_csv)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v)/1e3:.1f} | {sum(v)/tot:.3f} |")
traffic = {}
for rep in reps:
    lines += ["", f"## `--set full`: {os.path.basename(rep)}", ""]
    for d in full(rep):
        name = d["name"]
        base = name.split("(")[0].split("<")[0].replace("void ", "").strip()
        if base in PHASE and base not in traffic and "dram__bytes_read.sum" in d:
            b = sum(float(d[m][0].replace(",", "")) * SCALE.get(d[m][1], 1.0)
                    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
            traffic[base] = b / fpl
        lines.append(f"- **{d.pop('name')[:80]}**")
        for k, (v, u) in d.items():
            lines.append(f"  - {k}: {v} {u}")
print("\n".join(lines))
if traffic_out:
    import json
    phases = {}
    for k, v in traffic.items():
        phases[PHASE[k]] = phases.get(PHASE[k], 0.0) + v
    json.dump({"source": [os.path.basename(r) for r in reps], "frames_per_launch": fpl,
               "per_frame_bytes_by_kernel": traffic, "per_frame_bytes_by_phase": phases}, open(traffic_out, "w"), indent=1)
