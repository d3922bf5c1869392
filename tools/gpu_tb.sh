#!/bin/bash
# GPU round trip: build, the -m gpu suite (bounded), one bench line.  usage: bash tools/gpu_tb.sh TAG [pytest -k expr]
set -u
TAG=${1:-x}
K=${2:-}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1 || { tail -30 gpurun_out/build_$TAG.log; exit 1; }
if [ -n "$K" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -x -k "$K" > gpurun_out/tests_$TAG.log 2>&1
else
  timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/tests_$TAG.log 2>&1
fi
echo "tests rc=$?"; tail -15 gpurun_out/tests_$TAG.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - "$TAG" <<'PY'
import json, sys
tag = sys.argv[1]
try:
    d = json.load(open(f"gpurun_out/bench_{tag}.json"))
except Exception as e:
    print("bench failed", e); print(open(f"gpurun_out/bench_{tag}.err").read()[-3000:]); raise SystemExit
print("value", round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 3))
print({k: (round(v["ms_per_launch"], 3), round(v.get("tflops", 0), 2)) for k, v in d["kernels"].items()})
print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")}, "clocks", d["clocks"])
PY
