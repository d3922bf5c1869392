#!/bin/bash
# ncu --set full of the sweep + pcg kernels of one bench step (config 3); report in gpurun_out/$1.ncu-rep
R=${1:-sweep}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 || { tail gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"sweep|pcg_kernel" -s 3 -c 3 -o gpurun_out/$R $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
