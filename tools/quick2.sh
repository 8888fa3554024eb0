#!/bin/bash
T=${1:-q}
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo rc=$? >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers.log 2>&1
bash tools/quick.sh $T
