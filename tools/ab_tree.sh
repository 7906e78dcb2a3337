#!/bin/bash
# Prepare: rm -rf ab_old && mkdir ab_old && git archive <commit> | tar -x -C ab_old && make -C ab_old/paper_2501_02625_b200
mkdir -p gpurun_out
for r in 1 2 3; do
  for v in old new; do
    if [ $v = old ]; then d=ab_old; else d=.; fi
    (cd $d && timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
h=d['hbm_kernels']
print('$v', round(d['ms_per_step'],4), 'gemm', d['roofline']['per_step_ms'], 'k1', h['k1_rows_fwht_quant']['ms_per_step'], 'k2', h['k2_cols_fwht_quant']['ms_per_step'], 'k4', h['k4_unrotate']['ms_per_step'], 'glue', h['glue']['ms_per_step'], d['clocks']['sm_mhz'])")
  done
done
