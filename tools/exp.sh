#!/bin/bash
mkdir -p gpurun_out
for m in 0 7; do
HALO_GEMM_DEBUG_SKIP_EPI=$m timeout 200 python tools/bench_kernels.py gemm_sweep > gpurun_out/kern$m.log 2>&1
done
echo done
