#!/bin/bash
# Build, optionally run the GPU tests, then a bench run; prints a compact summary.
# usage (under gpurun): bash tools/gpu_quick.sh [tests] [bench-args...]
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
if [ "${1:-}" = "tests" ]; then
  shift
  timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
  tail -4 gpurun_out/gpu_tests.log
fi
python bench.py --no-cpu-baseline "$@" > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
try:
    d = json.load(open("gpurun_out/bench.json"))
except Exception as e:
    print("bench failed", e); print(open("gpurun_out/bench.err").read()[-2000:]); raise SystemExit
print("value", round(d["value"], 1), d["unit"], "ms/step", round(d["ms_per_step"], 3), "e2e", round(d.get("e2e", {}).get("value", 0), 1))
print({k: (round(v["ms_per_launch"], 3), round(v.get("tflops", 0), 2)) for k, v in d["kernels"].items()})
print("roofline", {k: d["roofline"][k] for k in ("kernel", "achieved", "frac")}, "clocks", d["clocks"])
PY
