#!/bin/bash
# Design study: K5 register split (helper warps dec / consumer warps inc) x straight-line TL limit,
# rebuilt on the box.  usage: bash tools/k5_regs.sh "40 232 6" "24 240 6" "24 240 7"
set -u
F=paper_2605_02670_b200/csrc/sweep3_impl.cuh
cp $F /tmp/s3r.orig
for v in "$@"; do
  set -- $v
  cp /tmp/s3r.orig $F
  # only the recover kernel's pair (first occurrences)
  python - "$1" "$2" "$3" <<'PY'
import sys
p = "paper_2605_02670_b200/csrc/sweep3_impl.cuh"
s = open(p).read()
s = s.replace('setmaxnreg.dec.sync.aligned.u32 40;', 'setmaxnreg.dec.sync.aligned.u32 %s;' % sys.argv[1], 1)
s = s.replace('setmaxnreg.inc.sync.aligned.u32 232;', 'setmaxnreg.inc.sync.aligned.u32 %s;' % sys.argv[2], 1)
s = s.replace('constexpr int K5_SLMAX = 6;', 'constexpr int K5_SLMAX = %s;' % sys.argv[3])
open(p, "w").write(s)
PY
  python -m paper_2605_02670_b200.build > gpurun_out/k5r.log 2>&1 || { tail -5 gpurun_out/k5r.log; continue; }
  for c in lattice256 star; do
    timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --warmup 3 > /tmp/k5r.json 2>/tmp/k5r.err
    python -c "import json; d=json.load(open('/tmp/k5r.json')); print('regs $1/$2 slmax $3 $c', round(d['ms_per_step'],3), round(d['kernels']['recover']['ms_per_launch'],3))" || tail -3 /tmp/k5r.err
  done
done
cp /tmp/s3r.orig $F
