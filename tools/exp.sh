#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
HALO_GEMM_STORE_HINT=0 timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_h0.log 2>&1
timeout 300 python tools/bench_kernels.py gemm > gpurun_out/kern_h1.log 2>&1
for i in 1 2; do
HALO_GEMM_STORE_HINT=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_h0_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_h1_$i.log 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_gemm -c 9 --csv python tools/prof_step.py 1 > gpurun_out/gemm_dram_h1.csv 2>/dev/null
