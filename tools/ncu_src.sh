#!/bin/bash
# ncu --set full with source-level sampling of one kernel of the config-3 bench step, exported as
# the raw and source pages (CSV) for tools/ncu_stall.py.  usage: bash tools/ncu_src.sh TAG REGEX [CONFIG]
TAG=${1:-k5}; RX=${2:-sweep3_kernel}; CFG=${3:-lattice256}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$RX -c 1 -o gpurun_out/${TAG}_full \
  python bench.py --config $CFG --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu $TAG rc=$?"
ncu -i gpurun_out/${TAG}_full.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_src.csv 2>/dev/null
ncu -i gpurun_out/${TAG}_full.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ls -la gpurun_out/${TAG}_*
