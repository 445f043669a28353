#!/bin/bash
# final measurements of a round: every config's bench line, the reference arm, prep launch list
bash tools/bench_all.sh
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_prep.csv python tools/profile_prep.py c4 2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_prep.csv gpurun_out/launches_prep_summary.csv
