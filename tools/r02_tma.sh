#!/bin/bash
# TMA-store epilogue check: selftest numerics + per-layer perf with/without, engine A/B, parity tests
T=${1:-tma}
mkdir -p gpurun_out
LCB_MMARES=1 LCB_TMASTORE=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest_tma.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest_tma.log
LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_selftest.log
LCB_MMARES=1 LCB_TMASTORE=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers_tma.log 2>&1
LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/${T}_layers.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "resnet or full or fresh or graph or vgg" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
bash tools/ab1.sh ${T} LCB_NO_TMA_STORE
tail -3 gpurun_out/${T}_selftest_tma.log; grep -c FAIL gpurun_out/${T}_selftest_tma.log; paste <(grep perf gpurun_out/${T}_layers.log | cut -c1-110) <(grep perf gpurun_out/${T}_layers_tma.log | awk '{print $(NF-7), $(NF-6)}')
tail -2 gpurun_out/${T}_pytest.log
