#!/bin/bash
# Design study: unroll pragma on K5's generic step-pair loop, rebuilt on the box.  usage: bash tools/k5_pragma.sh "" "#pragma unroll 1" "#pragma unroll 2"
set -u
F=paper_2605_02670_b200/csrc/sweep3_impl.cuh
cp $F /tmp/s3p.orig
for v in "$@"; do
  cp /tmp/s3p.orig $F
  python - "$v" <<'PY'
import sys
p = "paper_2605_02670_b200/csrc/sweep3_impl.cuh"
s = open(p).read()
old = "                for (; tt + 1 < tend; tt += 2) {"
s = s.replace(old, "                " + sys.argv[1] + "\n" + old, 1)
open(p, "w").write(s)
PY
  python -m paper_2605_02670_b200.build > gpurun_out/k5p.log 2>&1 || { tail -5 gpurun_out/k5p.log; continue; }
  for c in lattice256 star; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/k5p.json 2>/tmp/k5p.err
    python -c "import json; d=json.load(open('/tmp/k5p.json')); print('[$v] $c', round(d['ms_per_step'],3), round(d['kernels']['recover']['ms_per_launch'],3))" || tail -3 /tmp/k5p.err
  done
done
cp /tmp/s3p.orig $F
