#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list, ncu full captures.
# Usage (from this container):
#   gpurun --timeout 2400 -- 'bash tools/gpu_run.sh [tests] [bench] [launches] [full]'
# Everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
what="${*:-tests bench launches full}"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
for w in $what; do
  case $w in
    tests)
      timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
      echo "smoke rc=$?" >> gpurun_out/smoke.log ;;
    bench)
      timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
    bench_fast)
      timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log ;;
    kern)
      timeout 600 python tools/bench_kernels.py > gpurun_out/kern.log 2>&1; echo "kern rc=$?" >> gpurun_out/kern.log ;;
    k1ab)
      timeout 600 python tools/bench_kernels.py k1 > gpurun_out/k1_fused.log 2>&1
      HALO_K1_FUSED=0 timeout 600 python tools/bench_kernels.py k1 > gpurun_out/k1_twophase.log 2>&1 ;;
    train)
      timeout 900 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/pytest_train.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_train.log
      timeout 600 python bench.py --config cfg5 --layers 4 --steps 3 --warmup 3 > gpurun_out/bench_cfg5_l4.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_cfg5_l4.log ;;
    cfg5)
      timeout 1200 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/bench_cfg5.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_cfg5.log
      timeout 1200 python bench.py --config cfg5 --ac --steps 5 --warmup 3 > gpurun_out/bench_cfg5_ac.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_cfg5_ac.log ;;
    prof_cfg5)
      timeout 600 python tools/prof_cfg5.py 4 > gpurun_out/prof_cfg5.log 2>&1 ;;
    glue)
      timeout 900 python -m pytest tests/test_gpu_glue.py tests/test_gpu_train.py tests/test_gpu_layer.py tests/test_cxx_api.py -x -q > gpurun_out/pytest_glue.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_glue.log ;;
    block)
      timeout 900 python tools/bench_block.py --steps 10 > gpurun_out/bench_block.log 2>&1
      echo "rc=$?" >> gpurun_out/bench_block.log ;;
    sweep_right)
      timeout 600 python tools/sweep_fwht.py right > gpurun_out/sweep_right_new.jsonl 2>&1
      HALO_K1_LB=0 timeout 600 python tools/sweep_fwht.py right > gpurun_out/sweep_right_old.jsonl 2>&1 ;;
    lb)
      timeout 900 python -m pytest tests/test_gpu_cols_lb.py tests/test_gpu_kernels.py -k "left or large or transform" -x -q > gpurun_out/pytest_lb.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_lb.log
      timeout 600 python tools/sweep_fwht.py left > gpurun_out/sweep_left_new.jsonl 2>&1
      HALO_K2_LB=0 timeout 600 python tools/sweep_fwht.py left > gpurun_out/sweep_left_old.jsonl 2>&1 ;;
    prof_lb)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cols_lb -s 2 -c 2 \
        -f -o gpurun_out/prof_lb python tools/bench_lb.py 8192 1024 1 > gpurun_out/prof_lb.log 2>&1
      ncu -i gpurun_out/prof_lb.ncu-rep --page raw --csv > gpurun_out/prof_lb.raw.csv 2>/dev/null ;;
    lbt)
      for bl in 512 1024 2048 4096; do timeout 300 python tools/bench_lb.py 8192 $bl; done > gpurun_out/lbt.log 2>&1 ;;
    prof_block)
      timeout 600 python tools/prof_block.py int8 > gpurun_out/prof_block_int8.log 2>&1
      timeout 600 python tools/prof_block.py bf16 > gpurun_out/prof_block_bf16.log 2>&1 ;;
    wide)
      timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_layer.py tests/test_gpu_base_dims.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pytest_wide.log 2>&1
      echo "pytest rc=$?" >> gpurun_out/pytest_wide.log
      timeout 600 python tools/sweep_fwht.py right > gpurun_out/sweep_right_wide.jsonl 2>&1
      HALO_K1_WIDE=0 timeout 600 python tools/sweep_fwht.py right > gpurun_out/sweep_right_nowide.jsonl 2>&1 ;;
    prof_wide)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_rows_v4|k_cols_lb' -s 4 -c 4 \
        -f -o gpurun_out/prof_wide python tools/prof_lb_kernels.py > gpurun_out/prof_wide.log 2>&1 ;;
    sweep)
      timeout 900 python tools/sweep_fwht.py > gpurun_out/sweep.jsonl 2>&1 ;;
    kern_v2)
      HALO_K1_VERSION=2 timeout 600 python tools/bench_kernels.py k1 > gpurun_out/kern_v2.log 2>&1 ;;
    prof_k1)
      timeout 600 ncu --set full --clock-control none -k regex:k_rows_v -s 4 -c 2 \
        -f -o gpurun_out/prof_k1 python tools/bench_kernels.py k1 --reps 1 > gpurun_out/prof_k1.log 2>&1 ;;
    prof_k2)
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cols_v -s 0 -c 6 \
        -f -o gpurun_out/prof_k2 python tools/prof_step.py 1 > gpurun_out/prof_k2.log 2>&1 ;;
    prof_gemm)
      timeout 600 ncu --set full --clock-control none -k regex:k_gemm -s 3 -c 3 \
        -f -o gpurun_out/prof_gemm python tools/bench_kernels.py gemm --reps 1 > gpurun_out/prof_gemm.log 2>&1 ;;
    cpuref_cfg1)
      # one host core, ~9 min: runs in the background while the GPU work proceeds
      (timeout 1500 taskset -c 0 python tools/cpu_ref_cfg1.py > gpurun_out/cpu_ref_cfg1.json 2> gpurun_out/cpu_ref_cfg1.err) &
      CPUREF_PID=$! ;;
    bench_fsdp)
      timeout 600 python bench.py --fsdp --no-cpu-baseline > gpurun_out/bench_fsdp.log 2>&1; echo "rc=$?" >> gpurun_out/bench_fsdp.log ;;
    bench_cfg1)
      timeout 600 python bench.py --config cfg1 > gpurun_out/bench_cfg1.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_cfg1.log ;;
    traffic)
      timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
        -k regex:k_gemm --csv --log-file gpurun_out/gemm_traffic.csv python tools/prof_step.py 1 > gpurun_out/traffic.log 2>&1
      echo "traffic rc=$?" >> gpurun_out/traffic.log ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_small.py \
          > gpurun_out/sanitize_$tool.log 2>&1
        echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.log
      done ;;
    launches)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file gpurun_out/launches.csv python tools/prof_step.py 2 > gpurun_out/launches.log 2>&1
      echo "launches rc=$?" >> gpurun_out/launches.log ;;
    full)
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 3 -c 3 \
        -f -o gpurun_out/prof_gemm python tools/prof_step.py 1 > gpurun_out/prof_gemm.log 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_rows|k_cols' -s 0 -c 6 \
        -f -o gpurun_out/prof_fwht python tools/prof_step.py 1 > gpurun_out/prof_fwht.log 2>&1 ;;
  esac
done
if [ -n "${CPUREF_PID:-}" ]; then wait $CPUREF_PID; fi
# keep reps small enough to travel back (64 MiB cap): export raw CSV, drop big reps
for r in gpurun_out/*.ncu-rep; do
  [ -f "$r" ] || continue
  ncu -i "$r" --page raw --csv > "${r%.ncu-rep}.raw.csv" 2>/dev/null
  if [ $(stat -c %s "$r") -gt 25000000 ]; then rm -f "$r"; fi
done
echo done
