#!/bin/bash
# A/B of two builds of the library on one box: in-tree libhalo_b200.so vs
# paper_2501_02625_b200/libhalo_b200_old.so (HALO_B200_LIB), interleaved
mkdir -p gpurun_out
OLD=$PWD/paper_2501_02625_b200/libhalo_b200_old.so
for r in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then export HALO_B200_LIB=$OLD; else unset HALO_B200_LIB; fi
    timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
h=d['hbm_kernels']
print('$v', round(d['ms_per_step'],4), 'k1', h['k1_rows_fwht_quant']['ms_per_step'], h['k1_rows_fwht_quant']['frac'], 'k2', h['k2_cols_fwht_quant']['ms_per_step'], h['k2_cols_fwht_quant']['frac'], d['clocks']['sm_mhz'])"
  done
done
