#!/bin/bash
mkdir -p gpurun_out
for blk in 512 2048; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --block $blk > gpurun_out/bench_blk$blk.log 2>&1
done
