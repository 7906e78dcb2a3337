#!/bin/bash
# same-box A/B of the RMSNorm kernels: the previous build (libhalo_b200_old.so) vs this tree
for i in 1 2; do
  echo "old:"; HALO_B200_LIB=paper_2501_02625_b200/libhalo_b200_old.so python tools/bench_norm.py 20
  echo "new:"; python tools/bench_norm.py 20
done
