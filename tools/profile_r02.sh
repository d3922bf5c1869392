#!/bin/bash
# Round-2 evidence: ncu launch list of the config-3 bench command, ncu --set full of the config-3
# hot kernels and of config 4's global PCG.  usage (under gpurun): bash tools/profile_r02.sh TAG
set -u
R=${1:-r02}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$R.log 2>&1 || exit 1
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/${R}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_launches.csv $CMD > gpurun_out/${R}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sweep|pcg_warp|assemble|noise" -s 5 -c 5 -o gpurun_out/${R}_full $CMD > gpurun_out/${R}_ncu_full.log 2>&1
CMD4="python bench.py --config rgg --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"pcg_global" -c 1 -o gpurun_out/${R}_rgg_pcg $CMD4 > gpurun_out/${R}_ncu_rgg.log 2>&1
echo done
