#!/bin/bash
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 1 2 3 4; do
  GRF_PCG_VARIANT=$v python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/b_v$v.json 2>&1
  python -c "import json; d=json.load(open('gpurun_out/b_v$v.json')); print($v, d['ms_per_step'], d['kernels']['pcg']['ms_per_launch'])"
done
GRF_PCG_VARIANT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
