#!/bin/bash
# every BASELINE config through bench.py (one JSON line each) -> gpurun_out/bench_<cfg>.json
for c in ${CONFIGS:-c4 c1 c3 c5m c5c c2}; do
  extra=""
  [ "$c" != "c1" ] && [ -z "$WITH_CPU" ] && extra="--no-cpu-baseline"
  timeout 900 python bench.py --config $c --steps ${STEPS:-5} --warmup 3 $extra > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
