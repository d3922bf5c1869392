set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "host" > gpurun_out/zc_tests.log 2>&1; tail -3 gpurun_out/zc_tests.log
for z in 1 0; do
for c in lattice256 star tadpole lattice1 rgg; do
  GRF_HOST_ZC=$z timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/zc${z}_$c.json 2> gpurun_out/zc${z}_$c.err
  python -c "import json; d=json.load(open('gpurun_out/zc${z}_$c.json')); print('zc=$z $c', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['value'],2), round(d['e2e'].get('ms_per_step',0),3))" || tail -3 gpurun_out/zc${z}_$c.err
done; done
