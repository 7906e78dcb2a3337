#!/bin/bash
# same-box A/B of the SwiGLU GEMM epilogue (HALO_MLP_GLU_EPI) on the cfg2 bench,
# plus the forward's kernel times under the library's profile counters
for e in 0 1 0 1 0 1; do
  HALO_MLP_GLU_EPI=$e timeout 600 python bench.py --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('glu_epi=$e', round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done
for e in 0 1; do
  HALO_MLP_GLU_EPI=$e ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv python tools/prof_step.py 2 2>/dev/null \
    | python -c "
import csv,sys,collections
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:]:
    print('$e', r[ki][:60], r[vi])
" > gpurun_out/ab_glu_launch_$e.txt
done
