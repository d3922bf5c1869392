set -u
F=paper_2605_02670_b200/csrc/noise.cu
cp $F /tmp/noise.orig
for c in 16 32 64 1024; do
  cp /tmp/noise.orig $F
  sed -i "s/const int64_t cap = (int64_t)g.n_sm \* 16;/const int64_t cap = (int64_t)g.n_sm * $c;/" $F
  python -m paper_2605_02670_b200.build > /dev/null 2>&1 || { echo build fail; continue; }
  python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.load(sys.stdin); print('cap $c', d['kernels']['noise']['ms_per_launch'])"
done
cp /tmp/noise.orig $F
