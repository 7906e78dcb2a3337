#!/bin/bash
mkdir -p gpurun_out
timeout 200 python tools/bench_kernels.py gemm_sweep gemm_epi > gpurun_out/kern.log 2>&1
timeout 600 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
echo done
