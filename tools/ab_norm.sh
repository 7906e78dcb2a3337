#!/bin/bash
# same-box A/B of the RMSNorm backward: the previous build (libhalo_b200_old.so) vs this tree
for i in 1 2; do
  echo "old:"; HALO_B200_LIB=paper_2501_02625_b200/libhalo_b200_old.so python tools/bench_norm.py 20
  echo "new:"; python tools/bench_norm.py 20
done
for lib in paper_2501_02625_b200/libhalo_b200_old.so paper_2501_02625_b200/libhalo_b200.so; do
HALO_B200_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:'k_rmsnorm_bwd|k_sum_rows' python tools/bench_norm.py 2 2>/dev/null \
  | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value')
for r in rows[1:5]: print('$lib'[-10:], r[ki][:50], r[vi])"
done
