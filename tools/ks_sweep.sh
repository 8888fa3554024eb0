#!/bin/bash
# Split-K floor sweep (LCB_KS_MIN_STEPS) on the R18 / R50 / R152 benches. tag = $1
T=${1:-ks}
mkdir -p gpurun_out
for V in 0 2 4 8 16; do
  LCB_KS_MIN_STEPS=$V timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18_$V.json 2> gpurun_out/${T}_r18_$V.err
  LCB_KS_MIN_STEPS=$V timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_r50_$V.json 2> gpurun_out/${T}_r50_$V.err
done
