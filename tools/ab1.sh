#!/bin/bash
# One-shot A/B of an engine env switch (R18 b256 + R50 b128), then the GPU tests:
#   tools/ab1.sh TAG VAR [tests]
T=${1:-ab}; V=${2:-LCB_NO_CONV_HEAD}
mkdir -p gpurun_out
for X in 0 1; do
  env $V=$X timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18_$X.json 2>gpurun_out/${T}_r18_$X.err
  env $V=$X timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_r50_$X.json 2>gpurun_out/${T}_r50_$X.err
done
if [ "$3" == "tests" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
fi
for f in gpurun_out/${T}_r*.json; do python -c "
import json,sys
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],4), 'nocache', round(d['no_cache']['value']), d['hit_rate'])
"; done
tail -2 gpurun_out/${T}_pytest.log 2>/dev/null
