#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/bench_kernels.py fp8 > gpurun_out/kern_fmt.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --fmt fp8 > gpurun_out/bench_fp8.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --fmt fp6 > gpurun_out/bench_fp6.log 2>&1
