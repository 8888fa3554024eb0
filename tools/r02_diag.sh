#!/bin/bash
# Diagnose the fused-lookup conv: A/B LCB_NO_CONV_HEAD on R18/R50, launch list without it,
# and one full ncu capture of the R18 block-1 tap conv (2nd tc_conv launch of a step).
T=${1:-r02c}
mkdir -p gpurun_out
for X in 0 1; do
  LCB_NO_CONV_HEAD=$X timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18_nch$X.json 2>gpurun_out/${T}_r18_nch$X.err
  LCB_NO_CONV_HEAD=$X timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_r50_nch$X.json 2>gpurun_out/${T}_r50_nch$X.err
done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
LCB_NO_CONV_HEAD=1 timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_r18_nch1.csv python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_conv -s 1 -c 1 -o gpurun_out/${T}_tapconv_r18 python tools/profile_step.py resnet18_cifar bf16x3 > gpurun_out/${T}_ncu.log 2>&1
ls -la gpurun_out | tail
