#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/peer_stress.log
for i in 1 2 3 4; do
timeout 300 python -m pytest tests/test_gpu_peer.py -q -x -k two_processes >> gpurun_out/peer_stress.log 2>&1; echo "rc=$?" >> gpurun_out/peer_stress.log
done
timeout 600 python bench.py --no-cpu-baseline --fsdp > gpurun_out/bench_peer.log 2>&1; echo "rc=$?" >> gpurun_out/bench_peer.log
