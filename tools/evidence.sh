#!/bin/bash
# Round evidence under one tag: bench lines for every config (+ the default command with the CPU
# baseline, and the reference arm), the ncu launch list of the default command, ncu --set full of
# the config-3 hot kernels and of config 4's global PCG, the GPU tests.  usage: bash tools/evidence.sh TAG
set -u
R=${1:-r02f}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$R.log 2>&1 || { tail -20 gpurun_out/build_$R.log; exit 1; }
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${R}_gpu.txt
(nproc; lscpu | grep -E "Model name|Socket|Thread|Core") > gpurun_out/${R}_host.txt 2>&1
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
for c in tadpole lattice1 lattice256 rgg star; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/${R}_bench_$c.json')); print('$c', round(d['value'],2), round(d['ms_per_step'],3), 'ms', {k: round(v['ms_per_launch'],3) for k,v in d.get('kernels',{}).items()}, 'e2e', round(d['e2e']['value'],2), 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/${R}_bench_$c.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sweep|pcg_warp|assemble|noise" -s 5 -c 5 -o gpurun_out/${R}_full $CMD > gpurun_out/${R}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"pcg_global" -c 1 -o gpurun_out/${R}_rgg_pcg python bench.py --config rgg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_rgg.log 2>&1
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/${R}_gpu_tests.log 2>&1; tail -2 gpurun_out/${R}_gpu_tests.log
echo done
