#!/bin/bash
# same-box A/B of the large-block left kernel: in-tree library vs libhalo_b200_old.so
mkdir -p gpurun_out
OLD=$PWD/paper_2501_02625_b200/libhalo_b200_old.so
for r in 1 2; do
  for v in old new; do
    if [ $v = old ]; then export HALO_B200_LIB=$OLD; else unset HALO_B200_LIB; fi
    for bl in 512 1024 2048 4096; do echo -n "$v "; timeout 300 python tools/bench_lb.py 8192 $bl 2>/dev/null | head -1; done
  done
done
