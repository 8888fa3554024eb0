#!/bin/bash
mkdir -p gpurun_out
for H in 0 1; do for D in 0 1 2 4 6 7; do for L in 0 1 3 7 8 9; do
  HV=""; [ $H = 1 ] && HV="LCB_HALO=1"
  echo "halo=$H dbg=$D layer=$L $(env $HV LCB_DBG=$D LCB_TSTORE=1 LCB_MMARES=1 timeout 60 ./tests/cuda/tc_selftest --one $L | grep perf)"
done; done; done > gpurun_out/d_dbg.log 2>&1
LCB_TSTORE=1 LCB_MMARES=1 timeout 120 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/d_trace.log 2>&1
LCB_HALO=1 LCB_TSTORE=1 LCB_MMARES=1 timeout 120 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/d_trace_halo.log 2>&1
