#!/bin/bash
# End-of-round evidence pass: tools/r02_final.sh TAG
#  - pytest -m gpu (every test listed), smoke()
#  - bench: default (R50 b128, CPU baseline), reference arm, R18 b256, C1 (reference simulate_model),
#    VGG-16 threshold sweep point, R152 b512 / b1
#  - ncu launch lists (time + DRAM bytes) for R18 / R50 + traffic files; in-graph layer times
#  - ncu --set full of the R50 step's top kernel (stage-1 conv3 + fused projection) and the R18 3x3 conv
T=${1:-r02f}
mkdir -p gpurun_out
nproc > gpurun_out/${T}_nproc.txt; nvidia-smi > gpurun_out/${T}_nvsmi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
timeout 600 python bench.py --config c1_mlp --steps 50 --warmup 5 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
timeout 600 python bench.py --config vgg16_cifar --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_vgg.json 2> gpurun_out/${T}_bench_vgg.err
timeout 900 python bench.py --config resnet152 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r152.json 2> gpurun_out/${T}_bench_r152.err
timeout 900 python bench.py --config resnet152 --batch 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r152_b1.json 2> gpurun_out/${T}_bench_r152_b1.err
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in resnet18_cifar resnet50; do
  timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv python tools/profile_step.py $c bf16x3 > /dev/null 2>&1
  python tools/traffic.py gpurun_out/${T}_launches_$c.csv gpurun_out/traffic_${c}_bf16x3.json > gpurun_out/${T}_launches_$c.txt 2>&1
  python tools/launch_table.py gpurun_out/${T}_launches_$c.csv > gpurun_out/${T}_launch_table_$c.txt 2>&1
  timeout 300 python tools/layer_times.py $c bf16x3 compact > gpurun_out/${T}_layer_times_$c.txt 2>&1
done
P="ncu --profile-from-start off --set full --clock-control none --import-source on"
timeout 300 $P -k regex:tc_conv -s 2 -c 1 -o gpurun_out/${T}_ncu_r50_conv3proj python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
timeout 300 $P -k regex:tc_conv -s 1 -c 1 -o gpurun_out/${T}_ncu_r18_conv python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 300 $P -k regex:tc_stem -c 1 -o gpurun_out/${T}_ncu_r50_stem python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
ls -la gpurun_out | grep ${T} | tail -40
