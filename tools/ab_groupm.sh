#!/bin/bash
# same-box A/B of the GEMM tile raster (GROUP_M M-tiles per B panel): 16 (tree) vs 8 / 32 side builds
for r in 1 2; do
for lib in paper_2501_02625_b200/libhalo_b200.so paper_2501_02625_b200/libhalo_b200_g8.so paper_2501_02625_b200/libhalo_b200_g32.so; do
  HALO_B200_LIB=$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | grep '^{' | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib'[-12:], round(d['ms_per_step'],4), round(d['roofline']['per_step_ms'],4), d['clocks']['sm_mhz'])"
done; done
