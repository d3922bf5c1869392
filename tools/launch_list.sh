#!/bin/bash
# ncu launch list (gpu__time_duration per kernel) of one short bench run; prints per-kernel mean us
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/plain.log 2>&1 || { tail gpurun_out/plain.log; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1
python - <<'PY'
import csv, collections
rows = list(csv.DictReader([l for l in open("gpurun_out/launches.csv") if not l.startswith("==")]))
t = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        t[r["Kernel Name"].split("(")[0][-60:]].append(float(r["Metric Value"]) / 1000)
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:60s} n={len(v):3d} mean={sum(v)/len(v):10.1f} us")
PY
