#!/bin/bash
# A/B an engine env switch on the R18 / R50 benches: tools/ab_env.sh TAG VAR
T=${1:-abenv}; V=${2:-LCB_NO_WPREFETCH}
mkdir -p gpurun_out
for i in 1 2; do
  for X in 0 1; do
    env $V=$X timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18_${X}_$i.json 2>/dev/null
    env $V=$X timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_r50_${X}_$i.json 2>/dev/null
  done
done
