#!/bin/bash
# GPU tests (-x) + tc_conv selftest + R18/R50 benches (50 steps): tools/r02_check.sh TAG
T=$1
mkdir -p gpurun_out
timeout 300 ./tests/cuda/tc_selftest > gpurun_out/${T}_selftest.log 2>&1; echo "selftest rc=$?" >> gpurun_out/${T}_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers --trace > gpurun_out/${T}_layers.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18.json 2>gpurun_out/${T}_r18.err
timeout 900 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r50.json 2>gpurun_out/${T}_r50.err
tail -3 gpurun_out/${T}_selftest.log; tail -2 gpurun_out/${T}_pytest.log; grep perf gpurun_out/${T}_layers.log
for f in gpurun_out/${T}_r18.json gpurun_out/${T}_r50.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],4), 'nocache', round(d['no_cache']['value']), d['hit_rate'])
"; done
