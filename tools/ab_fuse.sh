#!/bin/bash
# A/B of the fused SwiGLU+absmax variants on the cfg2 bench
mkdir -p gpurun_out
for cfg in "0 0" "1 0" "0 1" "1 1"; do
  set -- $cfg
  HALO_MLP_FUSE_FWD=$1 HALO_MLP_FUSE_GLUE=$2 timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 5 2>/dev/null | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('fwd=$1 bwd=$2', round(d['ms_per_step'],4), {k:(v.get('ms_per_step'),v.get('frac')) for k,v in d['hbm_kernels'].items()}, d['kernel_time_share'])
"
done
