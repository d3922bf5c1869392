#!/bin/bash
# Design study: config-3 step per PCG warp-group size (env GRF_PCG_WPS).  usage: bash tools/wps.sh 1 2 4
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in "$@"; do
  GRF_PCG_WPS=$k timeout 300 python bench.py --config ${CONFIG:-lattice256} --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/wps$k.json 2> gpurun_out/wps$k.err
  echo "wps $k rc=$?"
  python -c "import json; d=json.load(open('/tmp/wps$k.json')); print({k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['pcg']['iter_mean'])" || tail -n 5 gpurun_out/wps$k.err
done
