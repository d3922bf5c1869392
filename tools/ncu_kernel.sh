#!/bin/bash
# ncu --set full of the kernels matching a regex in one bench step of a config.
# usage: bash tools/ncu_kernel.sh TAG CONFIG REGEX COUNT [GRF_ABLATE]
TAG=${1:-x}; CFG=${2:-lattice256}; RX=${3:-sweep}; CNT=${4:-1}; AB=${5:-0}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
GRF_ABLATE=$AB timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -c $CNT -o gpurun_out/${TAG}_full \
  python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu $TAG rc=$?"; tail -2 gpurun_out/${TAG}_ncu.log
