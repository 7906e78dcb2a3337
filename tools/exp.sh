#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
timeout 300 python tools/bench_kernels.py fp8 > gpurun_out/kern.log 2>&1
timeout 300 python bench.py --fmt fp8 --no-cpu-baseline --no-e2e > gpurun_out/bench_fp8.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_i8.log 2>&1
echo done
