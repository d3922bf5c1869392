python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in "64,64,64,32,32" "32,64,64,64,32" "32,64,64,32,32,32" "48,64,64,48,32" "64,64,64,32,32"; do
  GRF_HOST_CHUNKS=$p python bench.py --no-cpu-baseline --steps 5 --warmup 3 --e2e-steps 20 > /tmp/cp.json 2>/tmp/cp.err
  python -c "import json; d=json.load(open('/tmp/cp.json')); e=d['e2e']; print('plan $p', round(e['ms_per_step'],3), e['step_ms'])" || tail -2 /tmp/cp.err
done
