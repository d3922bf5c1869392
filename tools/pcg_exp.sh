#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$1', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"; }
run base
GRF_DEBUG_NOGATHER=1 run nogather
GRF_DEBUG_NOWRITE=1 run nowrite
GRF_DEBUG_NOGATHER=1 GRF_DEBUG_NOWRITE=1 run neither
