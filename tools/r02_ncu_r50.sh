#!/bin/bash
# Round-2 R50 evidence pass: in-graph per-block times (compact) for R50/R18 and
# ncu --set full captures of the step's main kernel classes: tools/r02_ncu_r50.sh TAG
T=${1:-r02n}
mkdir -p gpurun_out
timeout 300 python tools/layer_times.py resnet50 bf16x3 compact > gpurun_out/${T}_layer_times_r50.txt 2>&1
timeout 300 python tools/layer_times.py resnet18_cifar bf16x3 compact > gpurun_out/${T}_layer_times_r18.txt 2>&1
P="ncu --profile-from-start off --set full --clock-control none --import-source on"
S="python tools/profile_step.py resnet50 bf16x3"
timeout 300 $P -k regex:tc_conv -s 2 -c 1 -o gpurun_out/${T}_conv3proj $S > /dev/null 2>&1
timeout 300 $P -k regex:tc_conv -s 1 -c 1 -o gpurun_out/${T}_conv3x3 $S > /dev/null 2>&1
timeout 300 $P -k regex:tc_stem -c 1 -o gpurun_out/${T}_stem $S > /dev/null 2>&1
timeout 300 $P -k regex:maxpool -c 1 -o gpurun_out/${T}_maxpool $S > /dev/null 2>&1
timeout 300 $P -k regex:wide_lookup -s 8 -c 1 -o gpurun_out/${T}_wide $S > /dev/null 2>&1
timeout 300 $P -k regex:tc_conv -s 30 -c 1 -o gpurun_out/${T}_deep $S > /dev/null 2>&1
ls -la gpurun_out/${T}_*
