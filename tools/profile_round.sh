#!/bin/bash
# Round evidence: bench line (with cpu_baseline), ncu launch list, ncu --set full of the hot kernels.
# usage (under gpurun): bash tools/profile_round.sh r01
R=${1:-r01}
set -u
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,memory.total --format=csv > gpurun_out/${R}_gpu.txt
lscpu | grep -E "Model name|^CPU\(s\)" > gpurun_out/${R}_host.txt; nproc >> gpurun_out/${R}_host.txt
python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${R}_bench_ref.json 2>> gpurun_out/${R}_bench.err
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"sweep|pcg_warp|assemble" -s 4 -c 4 -o gpurun_out/${R}_full $CMD > gpurun_out/${R}_ncu_full.log 2>&1
echo done
