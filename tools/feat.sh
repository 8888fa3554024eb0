#!/bin/bash
T=${1:-f}
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${T}_pytest.log
timeout 900 python bench.py --config vgg16_cifar --steps 20 --warmup 3 --sweep 0.5,0.6,0.7,0.8,0.9,0.95,0.99 > gpurun_out/${T}_sweep_vgg.json 2> gpurun_out/${T}_sweep_vgg.err
timeout 900 python bench.py --config vgg16_cifar --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_vgg.json 2> gpurun_out/${T}_bench_vgg.err
timeout 900 python bench.py --config resnet152 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_bench_r152.json 2> gpurun_out/${T}_bench_r152.err
timeout 900 python bench.py --config resnet152 --batch 1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_r152_b1.json 2> gpurun_out/${T}_bench_r152_b1.err
timeout 600 python bench.py --config c1_mlp --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err
