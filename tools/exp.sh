#!/bin/bash
mkdir -p gpurun_out
timeout 900 python tools/bench_block.py > gpurun_out/block.log 2>&1
echo done
