#!/bin/bash
# Build, bench the given configs (compact lines), optionally the GPU tests.
# usage (under gpurun): bash tools/gpu_cfgs.sh "lattice256 star rgg" [tests]
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
for c in $1; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],2), d['unit'], round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_launch'],3) for k,v in d.get('kernels',{}).items()}, 'e2e', round(d.get('e2e',{}).get('value',0),2), 'frac', round(d['roofline']['frac'],3))" 2>/dev/null || tail -n 4 gpurun_out/bench_$c.err
done
if [ "${2:-}" = "tests" ]; then
  timeout 1500 python -m pytest tests/ -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1
  tail -5 gpurun_out/gpu_tests.log
fi
