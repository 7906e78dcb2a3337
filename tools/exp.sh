#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for i in 1 2 3; do
HALO_PDL=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pdl0_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_pdl1_$i.log 2>&1
done
