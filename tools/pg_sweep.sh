#!/bin/bash
# design study: global PCG variants (NB, minBlocks) on config 4
set -u
F=paper_2605_02670_b200/csrc/pcg_global.cu
cp $F /tmp/pg_orig.cu
for v in "4 4" "2 4" "8 4" "4 3" "2 5"; do
  set -- $v
  cp /tmp/pg_orig.cu $F
  sed -i "s/^constexpr int NB = [0-9];/constexpr int NB = $1;/; s/__launch_bounds__(GT, [0-9]) pcg_global_kernel/__launch_bounds__(GT, $2) pcg_global_kernel/" $F
  python -m paper_2605_02670_b200.build > /dev/null 2>&1 || { echo "build failed $v"; continue; }
  timeout 600 python bench.py --config rgg --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > /tmp/pg.json 2>/dev/null
  python -c "import json; d=json.load(open('/tmp/pg.json')); print('NB=$1 minb=$2', round(d['kernels']['pcg']['ms_per_launch'],1), 'ms pcg', round(d['ms_per_step'],1), 'ms step')"
done
cp /tmp/pg_orig.cu $F
