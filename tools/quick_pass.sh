#!/bin/bash
mkdir -p gpurun_out
T=${1:-q}
timeout 60 ./tests/cuda/pipe_bench > gpurun_out/${T}_pipe.log 2>&1
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 LCB_HALO=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_halo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_halo.log
for H in 0 1; do for D in 0 7; do
  HV=""; [ $H = 1 ] && HV="LCB_HALO=1"
  echo "halo=$H dbg=$D"; env $HV LCB_DBG=$D LCB_TSTORE=1 LCB_MMARES=1 timeout 120 ./tests/cuda/tc_selftest --layers | grep perf
done; done > gpurun_out/${T}_layers.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50.json 2> gpurun_out/${T}_bench_r50.err
