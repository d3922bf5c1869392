#!/bin/bash
# ncu --set full of kernels matching $2 in one bench step (config 3): gpurun_out/$1.ncu-rep
R=$1; K=$2; shift 2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail gpurun_out/build.log; exit 1; }
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $*"
$CMD > gpurun_out/plain.log 2>&1 || { tail gpurun_out/plain.log; exit 1; }
ncu --set full --clock-control none --import-source on -k regex:"$K" -s 1 -c 1 -o gpurun_out/$R $CMD > gpurun_out/ncu_full.log 2>&1
tail -2 gpurun_out/ncu_full.log
