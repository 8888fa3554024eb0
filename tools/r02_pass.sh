#!/bin/bash
# Round-2 GPU pass: tag = $1. Stages chosen by $STAGES (default: all).
# tests   : pytest -m gpu (no -x: every failure listed) + smoke
# sanit   : compute-sanitizer memcheck / initcheck / synccheck / racecheck over smoke()
# bench   : bench.py default (R50 b128) + R18 b256 + reference arm
# launches: ncu launch lists (time + DRAM bytes) for R18 / R50 steps
T=${1:-r02}
S=${STAGES:-tests sanit bench launches}
mkdir -p gpurun_out
nproc > gpurun_out/${T}_nproc.txt
nvidia-smi > gpurun_out/${T}_nvsmi.txt 2>&1
has() { [[ " $S " == *" $1 "* ]]; }
if has tests; then
  timeout 1800 python -m pytest tests -m gpu -q -rA --durations=15 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${T}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${T}_smoke.log
fi
if has sanit; then
  for tool in memcheck initcheck synccheck racecheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_sanitizer_$tool.log 2>&1
    echo "sanitizer $tool rc=$?" >> gpurun_out/${T}_sanitizer_$tool.log
  done
fi
if has bench; then
  timeout 900 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
  timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${T}_bench_ref.json 2> gpurun_out/${T}_bench_ref.err
  timeout 600 python bench.py --config resnet18_cifar --steps 50 --warmup 5 > gpurun_out/${T}_bench_r18.json 2> gpurun_out/${T}_bench_r18.err
  timeout 600 python bench.py --config c1_mlp --steps 50 --warmup 5 > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
fi
if has launches; then
  M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
  for c in resnet18_cifar resnet50; do
    timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv python tools/profile_step.py $c bf16x3 > /dev/null 2>&1
    python tools/traffic.py gpurun_out/${T}_launches_$c.csv gpurun_out/traffic_${c}_bf16x3.json > gpurun_out/${T}_launches_$c.txt 2>&1
  done
fi
ls -la gpurun_out | tail -40
