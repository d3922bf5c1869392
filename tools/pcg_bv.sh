#!/bin/bash
# Design study: config-3 step per PCG vertex batch (env GRF_PCG_BV).  usage: bash tools/pcg_bv.sh 1 2 4
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in "$@"; do
  GRF_PCG_BV=$k timeout 300 python bench.py --config ${CONFIG:-lattice256} --no-cpu-baseline --no-e2e --steps 20 --warmup 5 > /tmp/bv$k.json 2> gpurun_out/bv$k.err
  python -c "import json; d=json.load(open('/tmp/bv$k.json')); print('bv $k', round(d['ms_per_step'],3), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['pcg']['iter_mean'])" || tail -n 5 gpurun_out/bv$k.err
done
