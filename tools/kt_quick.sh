#!/bin/bash
# ncu launch list of the timed graph launches with per-kernel instruction counts and DRAM bytes (tag $1)
TAG=$1; shift
A="python bench.py --steps 16 --warmup 3 --no-cpu --no-extra --e2e-steps 8 $*"
DET_PROFILE_RANGE=2 ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_ -c 200 --csv \
  --log-file gpurun_out/${TAG}_kt.csv $A > gpurun_out/${TAG}_kt.log 2>&1
python - <<PY
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/${TAG}_kt.csv")) if len(r)>10]
h=rows[0]; ki,mi,vi,ui=h.index("Kernel Name"),h.index("Metric Name"),h.index("Metric Value"),h.index("Metric Unit")
acc=collections.defaultdict(lambda: collections.defaultdict(list))
S={"byte":1,"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9,"ns":1e-3,"us":1,"ms":1e3}
for r in rows[1:]:
    try: acc[r[ki].split("(")[0]][r[mi]].append(float(r[vi].replace(",",""))*S.get(r[ui],1))
    except ValueError: pass
tot=0
for k,m in sorted(acc.items(), key=lambda kv:-sum(kv[1]["gpu__time_duration.sum"])):
    d=m["gpu__time_duration.sum"]; mean=sum(d)/len(d); tot+=mean
    g=lambda n: sum(m.get(n,[0]))/max(1,len(m.get(n,[0])))
    print(f"{k[:46]:46s} n={len(d):3d} {mean:8.1f} us {g('smsp__inst_executed.sum')/1e6:7.2f}M inst  rd {g('dram__bytes_read.sum')/1e6:7.1f} MB wr {g('dram__bytes_write.sum')/1e6:7.1f} MB  warps {g('sm__warps_active.avg.pct_of_peak_sustained_active'):4.1f}%")
print(f"sum per iteration-branch {tot:.1f} us")
PY
