#!/bin/bash
# Generic GPU pass: tag = $1. Results land in gpurun_out/$1_*.
T=${1:-x}
mkdir -p gpurun_out
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_staged.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_staged.log
LCB_TSTORE=1 LCB_MMARES=1 LCB_HALO=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_halo.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_halo.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers.log 2>&1
LCB_TSTORE=1 LCB_MMARES=1 LCB_HALO=1 timeout 300 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/${T}_layers_halo.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
LCB_NO_HALO=1 LCB_UNFUSED_LOOKUP=1 timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r18_old.json 2> gpurun_out/${T}_bench_r18_old.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50.json 2> gpurun_out/${T}_bench_r50.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r18.csv python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r50.csv python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
if [ -n "$NCU_LAYERS" ]; then
  for L in $NCU_LAYERS; do
    LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/${T}_ncu_l$L ./tests/cuda/tc_selftest --one $L > /dev/null 2>&1
  done
fi
true
