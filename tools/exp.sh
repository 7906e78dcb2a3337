#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2; do
HALO_GEMM_BF16_EXACT=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_exact$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_fast$i.log 2>&1
done
HALO_GEMM_BF16_EXACT=1 timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_gexact.log 2>&1
timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_gfast.log 2>&1
