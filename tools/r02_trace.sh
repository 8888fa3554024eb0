#!/bin/bash
# tc_conv self-test (numerics), per-layer timings with traces, and graphed per-block times
T=${1:-r02e}
mkdir -p gpurun_out
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/${T}_layers.log 2>&1
timeout 300 python tools/layer_times.py resnet50 bf16x3 compact > gpurun_out/${T}_lt_r50.txt 2>&1
timeout 300 python tools/layer_times.py resnet18_cifar bf16x3 compact > gpurun_out/${T}_lt_r18.txt 2>&1
grep -E "perf|FAIL|rc=" gpurun_out/${T}_selftest.log | tail -5
grep perf gpurun_out/${T}_layers.log
