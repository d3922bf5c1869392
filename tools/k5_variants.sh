#!/bin/bash
# Design study: K5 compile-time variants rebuilt on the box ("GLATE SLMAX" pairs).  usage: bash tools/k5_variants.sh "false 6" "true 7" ...
set -u
F=paper_2605_02670_b200/csrc/sweep3_impl.cuh
cp $F /tmp/s3.orig
for v in "$@"; do
  set -- $v
  sed -i "s/^constexpr bool K5_GLATE = [a-z]*;/constexpr bool K5_GLATE = $1;/; s/^constexpr int K5_SLMAX = [0-9]*;/constexpr int K5_SLMAX = $2;/" $F
  python -m paper_2605_02670_b200.build > gpurun_out/k5v.log 2>&1 || { tail -5 gpurun_out/k5v.log; continue; }
  for c in lattice256 star; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/k5v.json 2>/tmp/k5v.err
    python -c "import json; d=json.load(open('/tmp/k5v.json')); print('glate $1 slmax $2 $c', round(d['ms_per_step'],3), round(d['kernels']['recover']['ms_per_launch'],3))" || tail -3 /tmp/k5v.err
  done
done
cp /tmp/s3.orig $F
