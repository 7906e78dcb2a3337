#!/bin/bash
# launch list + full captures of the current kernels, one step of the cfg2 MLP
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches.csv python tools/prof_step.py 2 > gpurun_out/launches.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 9 -c 3 \
  -f -o gpurun_out/prof_gemm python tools/prof_step.py 2 > gpurun_out/prof_gemm.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:'k_rows_v4|k_cols_v3' -s 10 -c 6 \
  -f -o gpurun_out/prof_fwht python tools/prof_step.py 2 > gpurun_out/prof_fwht.log 2>&1
for r in gpurun_out/*.ncu-rep; do
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  if [ $(stat -c %s "$r") -gt 25000000 ]; then rm -f "$r"; fi
done
echo done
