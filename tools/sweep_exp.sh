#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/b.json')); print('$1', round(d['ms_per_step'],3), {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" || tail -5 gpurun_out/b.json; }
GRF_SWEEP_IB=8 run ib8
GRF_SWEEP_IB=16 run ib16
GRF_SWEEP_IB=32 run ib32
