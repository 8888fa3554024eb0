#!/bin/bash
# A/B of an env switch (R18 + R50), GPU tests (-x), and the R50 launch list: tools/r02_ab_prof.sh TAG VAR [tests]
T=$1; V=$2
bash tools/ab1.sh $T $V $3
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --profile-from-start off --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_launches_resnet50.csv python tools/profile_step.py resnet50 bf16x3 > /dev/null 2>&1
python tools/launch_table.py gpurun_out/${T}_launches_resnet50.csv > gpurun_out/${T}_launches_resnet50.txt 2>&1
grep -E "wide|total" gpurun_out/${T}_launches_resnet50.txt
