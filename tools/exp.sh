#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layer.py -q -x -k llama > gpurun_out/pytest_blk.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_blk.log
timeout 1500 python tools/bench_block.py > gpurun_out/block.jsonl 2> gpurun_out/block.err; echo "rc=$?" >> gpurun_out/block.err
