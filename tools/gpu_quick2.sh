#!/bin/bash
# Build; bench the given configs (compact); optional pytest -k filter.  usage: bash tools/gpu_quick2.sh "lattice256 star" [kfilter]
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for c in $1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > /tmp/b.json 2>/tmp/b.err
  python -c "import json; d=json.load(open('/tmp/b.json')); print('$c', round(d['ms_per_step'],3), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" || tail -3 /tmp/b.err
done
if [ -n "${2:-}" ]; then
  timeout 1200 python -m pytest tests/ -q -m gpu -x -k "$2" > gpurun_out/q2_tests.log 2>&1; tail -2 gpurun_out/q2_tests.log
fi
