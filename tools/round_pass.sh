#!/bin/bash
# Full measurement pass for the current tree: tag = $1 (results in gpurun_out/$1_*).
T=${1:-r}
mkdir -p gpurun_out
nvidia-smi > gpurun_out/${T}_nvsmi.txt 2>&1; nproc > gpurun_out/${T}_nproc.txt
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for c in resnet18_cifar resnet50; do
  timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv python tools/profile_step.py $c bf16x3 > /dev/null 2>&1
  python tools/traffic.py gpurun_out/${T}_launches_$c.csv gpurun_out/traffic_${c}_bf16x3.json > gpurun_out/${T}_launches_$c.txt 2>&1; cp gpurun_out/traffic_${c}_bf16x3.json profiles/
  timeout 300 python tools/step_roofline.py $c bf16x3 > gpurun_out/${T}_steps_$c.txt 2>&1
done
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
timeout 600 python bench.py --steps 30 --warmup 5 --precision bf16 --no-cpu-baseline > gpurun_out/${T}_bench_r18_bf16.json 2> gpurun_out/${T}_bench_r18_bf16.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r50.json 2> gpurun_out/${T}_bench_r50.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --precision bf16 --no-cpu-baseline > gpurun_out/${T}_bench_r50_bf16.json 2> gpurun_out/${T}_bench_r50_bf16.err
if [ -n "$NCU_FULL" ]; then
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:tc_conv -c 3 -o gpurun_out/${T}_ncu_tcconv_r18 python tools/profile_step.py resnet18_cifar bf16x3 > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"cache_head|rows_fc|gap_bins" -c 6 -o gpurun_out/${T}_ncu_lookup_r50 python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
fi
ls -la gpurun_out | tail -30
