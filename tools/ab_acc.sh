#!/bin/bash
# same-box A/B of dx = ex_gate + ex_up fused into the up projection's K4 store (HALO_MLP_ACC_DX)
for e in 0 1 0 1; do
  HALO_MLP_ACC_DX=$e timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('acc_dx=$e', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
for e in 0 1; do
  HALO_MLP_ACC_DX=$e ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_step.py 1 2>/dev/null | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
ks=[(r[ki][:40], float(r[vi])) for r in rows[1:] if 'halo_b200' in r[ki]]
print('acc_dx=$e', 'ours total us', round(sum(v for _,v in ks)/1e3,1), 'last 4:', [(k[:24], v) for k,v in ks[-4:]])"
done
