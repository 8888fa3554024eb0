#!/bin/bash
# Generic GPU pass: tag = $1. Results land in gpurun_out/$1_*.
T=${1:-x}
mkdir -p gpurun_out
[ -x tests/cuda/umma_shift_test ] && for v in 0 1 2 3; do timeout 60 ./tests/cuda/umma_shift_test $v; done > gpurun_out/${T}_umma_shift.log 2>&1
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_tstore.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_tstore.log
timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers.log 2>&1
LCB_TSTORE=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers_tstore.log 2>&1
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_mmares.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_mmares.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers_mmares.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50.json 2> gpurun_out/${T}_bench_r50.err
LCB_NO_MMA_RESIDUAL=1 timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50_nomma.json 2> gpurun_out/${T}_bench_r50_nomma.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r18.csv python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r50.csv python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
true
