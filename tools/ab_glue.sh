#!/bin/bash
# A/B of the fused block glue on one box (HALO_BLOCK_UNFUSED_GLUE)
mkdir -p gpurun_out
for u in 1 0 1 0; do
  HALO_BLOCK_UNFUSED_GLUE=$u timeout 600 python bench.py --config cfg5 --layers 8 --steps 4 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('unfused=$u', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
