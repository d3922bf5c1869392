#!/bin/bash
# Design study: config-4 step per global-PCG variant (env GRF_PCGV).  usage: bash tools/pcgv.sh 0 1 2 ...
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in "$@"; do
  GRF_PCGV=$k timeout 600 python bench.py --config ${CONFIG:-rgg} --no-cpu-baseline --no-e2e --steps 3 --warmup 1 > /tmp/pcgv$k.json 2> gpurun_out/pcgv$k.err
  echo "pcgv $k rc=$?"
  python -c "import json; d=json.load(open('/tmp/pcgv$k.json')); print({k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()}, d['pcg'])" || tail -n 5 gpurun_out/pcgv$k.err
done
