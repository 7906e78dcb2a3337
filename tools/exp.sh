#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --fmt fp8 --no-cpu-baseline > gpurun_out/bench_fp8.log 2>&1
timeout 900 python bench.py --fmt fp6 --no-cpu-baseline > gpurun_out/bench_fp6.log 2>&1
timeout 900 python bench.py --block 0 --no-cpu-baseline --no-e2e > gpurun_out/bench_blk0.log 2>&1; echo "rc=$?" >> gpurun_out/bench_blk0.log
