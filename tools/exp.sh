#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pp.log 2>&1; echo "rc=$?" >> gpurun_out/bench_pp.log
