timeout 300 ./tests/cuda/tc_selftest > gpurun_out/h_selftest.log 2>&1; echo rc=$? >> gpurun_out/h_selftest.log
LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/h_layers.log 2>&1
LCB_DBG=7 LCB_TSTORE=1 LCB_MMARES=1 timeout 300 ./tests/cuda/tc_selftest --layers > gpurun_out/h_layers_d7.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/h_pytest.log 2>&1
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/h_bench_r18.json 2> gpurun_out/h_bench_r18.err
timeout 900 python bench.py --config resnet50 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/h_bench_r50.json 2> gpurun_out/h_bench_r50.err
