#!/bin/bash
# same-box A/B of programmatic dependent launch (HALO_PDL)
for r in 1 2 3; do
  for p in 1 0; do
    HALO_PDL=$p timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
h=d['hbm_kernels']
print('pdl=$p', round(d['ms_per_step'],4), 'gemm', d['roofline']['per_step_ms'], 'k1', h['k1_rows_fwht_quant']['ms_per_step'], 'k2', h['k2_cols_fwht_quant']['ms_per_step'], d['clocks']['sm_mhz'])"
  done
done
