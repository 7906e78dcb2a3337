#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_mlp.py -q -x > gpurun_out/pytest_mlp.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_mlp.log
for i in 1 2; do
HALO_MLP_FUSE_FWD=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ff0_$i.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_ff1_$i.log 2>&1
done
