#!/bin/bash
# ncu --set full of the sweep2 kernels (condense + recover) of one config-3 bench step.  usage: bash tools/ncu_sweep2.sh TAG
TAG=${1:-x}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep2 -c 2 -o gpurun_out/${TAG}_full python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
tail -3 gpurun_out/${TAG}_ncu.log
