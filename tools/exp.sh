#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HALO_GEMM_SPLITK=0 timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_sk0.log 2>&1
timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_sk1.log 2>&1
for i in 1 2; do
HALO_GEMM_SPLITK=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_sk0_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_sk1_$i.log 2>&1
done
