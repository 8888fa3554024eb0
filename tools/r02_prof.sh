#!/bin/bash
# launch list of one compact step + full ncu capture of one kernel: tools/r02_prof.sh TAG CONFIG KERNEL_REGEX SKIP
T=${1:-r02g}; C=${2:-resnet50}; K=${3:-wide_lookup}; S=${4:-3}
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_$C.csv python tools/profile_step.py $C bf16x3 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${T}_launches_$C.csv > gpurun_out/${T}_launches_$C.txt 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:$K -s $S -c 1 -o gpurun_out/${T}_$K python tools/profile_step.py $C bf16x3 > gpurun_out/${T}_ncu.log 2>&1
timeout 300 python tools/layer_times.py $C bf16x3 compact > gpurun_out/${T}_lt_$C.txt 2>&1
tail -3 gpurun_out/${T}_ncu.log; cat gpurun_out/${T}_lt_$C.txt
