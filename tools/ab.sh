#!/bin/bash
# A/B: parity suite, then R18/R50 bench with and without programmatic dependent launch. tag = $1
T=${1:-ab}
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo rc=$? >> gpurun_out/${T}_selftest.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest.log 2>&1
for V in 0 1; do
LCB_NO_PDL=$V timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r18_nopdl$V.json 2> gpurun_out/${T}_bench_r18_nopdl$V.err
LCB_NO_PDL=$V timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50_nopdl$V.json 2> gpurun_out/${T}_bench_r50_nopdl$V.err
done
