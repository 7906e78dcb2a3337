#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline --no-e2e --graph > gpurun_out/bench_graph.log 2>&1; echo "rc=$?" >> gpurun_out/bench_graph.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --fmt fp6 > gpurun_out/bench_fp6.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fp6.log
