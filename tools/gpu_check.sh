#!/bin/bash
# One GPU-box pass: parity suite, bench lines, launch list, full ncu of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
cp -f MEASURED_PEAKS.json gpurun_out/ 2>/dev/null
nproc > gpurun_out/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_r18.json 2> gpurun_out/bench_r18.err
timeout 600 python bench.py --steps 30 --warmup 5 --precision bf16 --no-cpu-baseline > gpurun_out/bench_r18_bf16.json 2> gpurun_out/bench_r18_bf16.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_r50.json 2> gpurun_out/bench_r50.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r18_bf16x3.csv python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/launches.log 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_conv -c 3 -o gpurun_out/prof_tcconv_r18 python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"pool|cache_head|exit_compact" -c 6 -o gpurun_out/prof_lookup_r18 python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/ncu_lookup.log 2>&1
ls -la gpurun_out
