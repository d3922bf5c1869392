#!/bin/bash
# One bench line per BASELINE config (plus config 4 edge-partitioned) into gpurun_out/bench_<tag>_<config>.json
set -u
TAG=${1:-r02}
shift || true
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for c in ${@:-tadpole lattice1 lattice256 rgg star}; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_${TAG}_$c.json 2> gpurun_out/bench_${TAG}_$c.err
  echo "$c rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_${TAG}_$c.json')); print(round(d['value'],2), d['unit'], round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_launch'],3) for k,v in d.get('kernels',{}).items()}, 'e2e', round(d.get('e2e',{}).get('value',0),2), 'graph', d.get('run',{}).get('cuda_graph'))" 2>/dev/null || tail -n 4 gpurun_out/bench_${TAG}_$c.err
done
