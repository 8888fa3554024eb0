#!/bin/bash
# r01b: parity after the batched-head change, R50 bench, deep-layer tc_conv capture.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r50_bf16x3.csv python tools/profile_step.py resnet50 bf16x3 > gpurun_out/launches50.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_conv -s 15 -c 5 -o gpurun_out/prof_tcconv_r18_deep python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/ncu_deep.log 2>&1
ls -la gpurun_out
