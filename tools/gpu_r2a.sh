set -u
free -g > gpurun_out/r02_host_mem.txt; nproc >> gpurun_out/r02_host_mem.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "config4 or config5 or long_edges" --durations=10 > gpurun_out/r02_newparity.log 2>&1
tail -15 gpurun_out/r02_newparity.log
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02_bench0.json 2> gpurun_out/r02_bench0.err
python -c "import json; d=json.load(open('gpurun_out/r02_bench0.json')); print(d['value'], d['ms_per_step'], {k:round(v['ms_per_launch'],3) for k,v in d['kernels'].items()})"
