#!/bin/bash
# per-kernel launch list of ONE device step (ncu, serialized, cold-cache): gpurun_out/launches_<cfg>.csv
cfg=${1:-c4}
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --csv --log-file gpurun_out/launches_$cfg.csv python tools/profile_step.py $cfg \
    > gpurun_out/ncu_$cfg.log 2>&1
echo "ncu $cfg rc=$?"
python tools/launch_summary.py gpurun_out/launches_$cfg.csv gpurun_out/launches_${cfg}_summary.csv
head -30 gpurun_out/launches_${cfg}_summary.csv
