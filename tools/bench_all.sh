#!/bin/bash
# every BASELINE config through bench.py (one JSON line each) -> gpurun_out/bench_<cfg>.json
# steps per config sized so the timed region spans >= ~0.5 s (clocks sampled every 50 ms)
declare -A STEPS=([c1]=300 [c3]=100 [c4]=20 [c5m]=20 [c5c]=20 [c2]=5)
for c in ${CONFIGS:-c4 c1 c3 c5m c5c c2}; do
  timeout 900 python bench.py --config $c --steps ${STEPS[$c]} --warmup 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
