#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1200 python tools/sweep_fwht.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
