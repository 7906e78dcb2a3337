#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer.py -x -q > gpurun_out/pytest_peer.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_peer.log
timeout 600 python bench.py --no-cpu-baseline --fsdp > gpurun_out/bench_peer.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_peer.log
