#!/bin/bash
# Design study: K5 (sweep3_kernel) steps per stage IBK, rebuilt on the box per value.
# usage: bash tools/k5_ibk.sh 8 10 12
set -u
F=paper_2605_02670_b200/csrc/sweep3_impl.cuh
cp $F /tmp/sweep3_impl.cuh.orig
for k in "$@"; do
  sed -i "s/^constexpr int IBK = [0-9]*;/constexpr int IBK = $k;/" $F
  python -m paper_2605_02670_b200.build > gpurun_out/ibk_build_$k.log 2>&1 || { tail -5 gpurun_out/ibk_build_$k.log; continue; }
  for c in ${CONFIGS:-lattice256 star}; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/ibk$k$c.json 2> gpurun_out/ibk$k$c.err
    python -c "import json; d=json.load(open('/tmp/ibk$k$c.json')); print('ibk $k $c', round(d['ms_per_step'],3), {k: round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})" || tail -n 3 gpurun_out/ibk$k$c.err
  done
done
cp /tmp/sweep3_impl.cuh.orig $F
