#!/bin/bash
# same-box A/B of the residual add in the down projection's epilogue (HALO_MLP_RES_EPI) on cfg5, 8 layers
for e in 0 1 0 1; do
  HALO_MLP_RES_EPI=$e timeout 600 python bench.py --config cfg5 --layers 8 --steps 4 --warmup 3 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('res_epi=$e', round(d['ms_per_step'],2), d['clocks']['sm_mhz'])"
done
