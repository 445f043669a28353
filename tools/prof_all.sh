set -x
for c in c1 c3 c4 c5m c5c c2; do timeout 900 bash tools/launches.sh $c > /dev/null 2>&1; echo "$c $?"; done
python tools/traffic_from_launches.py gpurun_out/r2_traffic.json c1=gpurun_out/launches_c1.csv c3=gpurun_out/launches_c3.csv c4=gpurun_out/launches_c4.csv c5m=gpurun_out/launches_c5m.csv c5c=gpurun_out/launches_c5c.csv c2=gpurun_out/launches_c2.csv > /dev/null
timeout 600 ncu --set full --import-source on --clock-control none -k regex:tc_scan_kernel -s 3 -c 1 -o gpurun_out/tc_c4_final python tools/profile_step.py c4 > gpurun_out/ncu_tc_final.log 2>&1; echo "tc $?"
timeout 300 ncu --set full --import-source on --clock-control none -k regex:small_screened -c 1 -o gpurun_out/small_c1_final python tools/small_run.py c1 1 > gpurun_out/ncu_small_final.log 2>&1; echo "small $?"
