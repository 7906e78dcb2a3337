for lib in paper_2501_02625_b200/libhalo_b200_old.so paper_2501_02625_b200/libhalo_b200.so; do
  echo $lib; HALO_B200_LIB=$lib python tools/bench_norm.py 20
  HALO_B200_LIB=$lib ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:'k_rmsnorm_bwd|k_sum_rows' python tools/bench_norm.py 1 2>/dev/null \
  | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; ki=h.index('Kernel Name'); vi=h.index('Metric Value'); mi=h.index('Metric Name')
for r in rows[1:5]: print('  ', r[ki][:40], r[mi], r[vi])"
done
