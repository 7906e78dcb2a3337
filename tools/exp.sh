#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -rs > gpurun_out/pytest_fuzz.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_fuzz.log
