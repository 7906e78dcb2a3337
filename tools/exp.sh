#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
HALO_K2_TMA=0 timeout 300 python tools/bench_kernels.py k2 > gpurun_out/kern_k2.log 2>&1
echo TMA >> gpurun_out/kern_k2.log
timeout 300 python tools/bench_kernels.py k2 >> gpurun_out/kern_k2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
