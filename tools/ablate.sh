#!/bin/bash
# Design study: time the config-3 step with the sweep2 kernels' ablation bits (env GRF_ABLATE;
# results are wrong by construction).  usage: bash tools/ablate.sh 0 1 2 4 ...
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for k in "$@"; do
  GRF_ABLATE=$k timeout 300 python bench.py --config ${CONFIG:-lattice256} --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/abl$k.json 2> gpurun_out/abl$k.err
  echo "ablate $k rc=$?"
  python -c "import json; d=json.load(open('/tmp/abl$k.json')); print({k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" || tail -n 5 gpurun_out/abl$k.err
done
