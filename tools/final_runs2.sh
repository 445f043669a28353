#!/bin/bash
# end-of-round batch: GPU tests, smoke, every config's bench line, reference arm, launch
# lists (C4, C3, C5m), one ncu --set full capture of the C4 tensor-core scan
timeout 1500 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/final_gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
bash tools/final_runs.sh
for c in c4 c3 c5m c1; do timeout 900 bash tools/launches.sh $c > /dev/null 2>&1; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o gpurun_out/tc_c4_final2 python tools/profile_step.py c4 > gpurun_out/ncu_tc_final2.log 2>&1
