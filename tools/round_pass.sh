#!/bin/bash
# Full measurement pass for the current tree: tag = $1 (results in gpurun_out/$1_*).
T=${1:-r}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_nvsmi.txt 2>&1; nproc > gpurun_out/${T}_nproc.txt
cp -f MEASURED_PEAKS.json gpurun_out/${T}_peaks.json 2>/dev/null
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
timeout 600 python bench.py --steps 30 --warmup 5 --precision bf16 --no-cpu-baseline > gpurun_out/${T}_bench_r18_bf16.json 2> gpurun_out/${T}_bench_r18_bf16.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50.json 2> gpurun_out/${T}_bench_r50.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --precision bf16 --no-cpu-baseline > gpurun_out/${T}_bench_r50_bf16.json 2> gpurun_out/${T}_bench_r50_bf16.err
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers.log 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r18.csv python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_r50.csv python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_conv -c 3 -o gpurun_out/${T}_ncu_tcconv_r18 python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gap|pool|cache_head|exit|logits" -c 8 -o gpurun_out/${T}_ncu_lookup_r50 python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
fi
ls -la gpurun_out | tail -30
