#!/bin/bash
mkdir -p gpurun_out
LCB_DBG=7 LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/m_l3_d7 ./tests/cuda/tc_selftest --one 3 > gpurun_out/m_ncu.log 2>&1
LCB_DBG=0 LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/m_l3_d0 ./tests/cuda/tc_selftest --one 3 >> gpurun_out/m_ncu.log 2>&1
LCB_DBG=0 LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_conv -s 3 -c 1 -o gpurun_out/m_l0_d0 ./tests/cuda/tc_selftest --one 0 >> gpurun_out/m_ncu.log 2>&1
