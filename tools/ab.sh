#!/bin/bash
# A/B: quick_perf scan_ms under NNM_TC_DBG settings, alternated on the same box
for rep in 1 2; do for m in "$@"; do
  NNM_TC_DBG=$m timeout 300 python tools/quick_perf.py ${SHAPE:-2000000x25x4000} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('dbg=$m scan_ms=%.1f total_ms=%.1f replay=%.1f' % (r['scan_ms'], r['total_ms'], r['replay_ms']))"
done; done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv,noheader
