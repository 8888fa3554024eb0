#!/bin/bash
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/i_l7_direct ./tests/cuda/tc_selftest --one 7 > gpurun_out/i_ncu1.log 2>&1
LCB_TSTORE=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/i_l7_tstore ./tests/cuda/tc_selftest --one 7 > gpurun_out/i_ncu2.log 2>&1
LCB_MMARES=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/i_l9_mmares ./tests/cuda/tc_selftest --one 9 > gpurun_out/i_ncu3.log 2>&1
timeout 300 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_stem -c 1 -o gpurun_out/i_stem python tools/profile_step.py resnet50 bf16x3 > gpurun_out/i_ncu4.log 2>&1
ls -la gpurun_out/i_*
