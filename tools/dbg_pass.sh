#!/bin/bash
# Bottleneck isolation (tc_conv debug bits) on layer configs of tests/cuda/tc_selftest --one:
# 0 r18 b1 3x3 64, 3 r18 16x16 128, 7 r50 1x1 64->64, 9 r50 1x1 64->256 res
mkdir -p gpurun_out
for H in 0 1; do for D in 0 1 2 4 3 5 6 7; do for L in 0 3 7 9; do
  HV=""; [ $H = 1 ] && HV="LCB_HALO=1"
  echo "halo=$H dbg=$D layer=$L $(env $HV LCB_DBG=$D LCB_TSTORE=1 LCB_MMARES=1 timeout 60 ./tests/cuda/tc_selftest --one $L | grep perf)"
done; done; done > gpurun_out/l_dbg.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/l_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/l_pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/l_bench_r18.json 2> gpurun_out/l_bench_r18.err
LCB_NO_HALO=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/l_bench_r18_nohalo.json 2> gpurun_out/l_bench_r18_nohalo.err
LCB_NO_HALO=1 LCB_UNFUSED_LOOKUP=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/l_bench_r18_old.json 2> gpurun_out/l_bench_r18_old.err
