F=paper_2605_02670_b200/csrc/pcg.cu
cp $F /tmp/pcg.orig
for v in 32 64 16; do
  cp /tmp/pcg.orig $F
  sed -i "s/constexpr int ASM_VB = 32;/constexpr int ASM_VB = $v;/" $F
  python -m paper_2605_02670_b200.build > /dev/null 2>&1 || { echo build fail; continue; }
  python bench.py --no-cpu-baseline --no-e2e --steps 10 --warmup 3 | python -c "import json,sys; d=json.load(sys.stdin); print('asm_vb $v', d['ms_per_step'], d['kernels']['pcg']['ms_per_launch'])"
done
cp /tmp/pcg.orig $F
