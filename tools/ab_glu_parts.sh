#!/bin/bash
# where the SwiGLU epilogue's time goes: launch durations of the up GEMM with
# the g loads (8) or the silu math (9) removed
# (timing experiments only)
for d in 0 8 9; do
  HALO_GEMM_DEBUG_SKIP_EPI=$d ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv python tools/prof_step.py 1 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
print('dbg=$d', [r[vi] for r in rows[1:] if 'k_gemm' in r[ki] or 'swiglu_fwd' in r[ki]][:3])
"
done
