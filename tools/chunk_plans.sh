#!/bin/bash
# Design study: config-3 e2e per grf_sample_host chunk plan (env GRF_HOST_CHUNKS) and direct last chunk (GRF_HOST_ZC)
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for z in 1 2; do
for p in "64,64,64,32,32" "96,96,32,32" "128,64,32,32" "64,64,64,64" "96,64,64,32" "80,80,64,32" "112,80,32,32" "128,96,32" "160,64,32" "192,32,32"; do
  GRF_HOST_ZC=$z GRF_HOST_CHUNKS=$p timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > /tmp/cp.json 2>/tmp/cp.err
  python -c "import json; d=json.load(open('/tmp/cp.json')); print('zc=$z plan $p', 'e2e ms', round(d['e2e']['ms_per_step'],3))" || tail -2 /tmp/cp.err
done; done
