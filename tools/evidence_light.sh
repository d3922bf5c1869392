#!/bin/bash
# Bench lines for every config (+ the default command with the CPU baseline, the reference arm) and
# the ncu launch list of the default command; no full captures (tools/evidence.sh has those).
# usage: bash tools/evidence_light.sh TAG
set -u
R=${1:-r02i}
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,clocks.sm,power.limit --format=csv > gpurun_out/${R}_gpu.txt
(nproc; lscpu | grep -E "Model name|Socket|Thread|Core") > gpurun_out/${R}_host.txt 2>&1
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
for c in tadpole lattice1 lattice256 rgg star; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/${R}_bench_$c.json 2> gpurun_out/${R}_bench_$c.err
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
CMD1="python bench.py --config lattice1 --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches_lattice1.csv $CMD1 > gpurun_out/${R}_ncu_launch1.log 2>&1
echo done
