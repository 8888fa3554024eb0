#!/bin/bash
mkdir -p gpurun_out
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/selftest.log 2>&1; echo "rc=$?" >> gpurun_out/selftest.log
timeout 300 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/layers.log 2>&1; echo "rc=$?" >> gpurun_out/layers.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r18_bf16x3.csv python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/launches.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_bf16x3.csv python tools/profile_step.py resnet50 bf16x3 > gpurun_out/launches50.log 2>&1
