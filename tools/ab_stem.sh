#!/bin/bash
# Stem epilogue sets A/B (LCB_STEM_EPI_SETS=1: one set of 8 epilogue warps; default 2):
# smoke + GPU tests, stem launch times (ncu, one kernel), R50/R18/VGG benches, alternating.
T=${1:-abstem}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest.log
for X in 2 1; do
  for c in resnet50 resnet18_cifar; do
    LCB_STEM_EPI_SETS=$X timeout 600 ncu --profile-from-start off -k regex:tc_stem --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${T}_ncu_${c}_$X.csv python tools/profile_step.py $c bf16x3 > /dev/null 2>&1
  done
done
for i in 1 2; do
  for X in 2 1; do
    LCB_STEM_EPI_SETS=$X timeout 900 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r50_${X}_$i.json 2>/dev/null
    LCB_STEM_EPI_SETS=$X timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_r18_${X}_$i.json 2>/dev/null
    LCB_STEM_EPI_SETS=$X timeout 600 python bench.py --config vgg16_cifar --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_vgg_${X}_$i.json 2>/dev/null
  done
done
LCB_STEM_EPI_SETS=2 timeout 300 python tools/layer_times.py resnet50 bf16x3 compact > gpurun_out/${T}_layer_times_r50.txt 2>&1
for f in gpurun_out/${T}_*.json; do python -c "
import json
d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['ms_per_step'],4), 'nocache', round(d['no_cache']['value']))
"; done
for f in gpurun_out/${T}_ncu_*.csv; do echo $f; grep tc_stem $f | awk -F'","' '{print $(NF-2), $NF}' | head -8; done
tail -2 gpurun_out/${T}_pytest.log gpurun_out/${T}_smoke.log
