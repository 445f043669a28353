#!/bin/bash
# per-item time of the TC scan under the NNM_TC_DBG timing experiments (2M x 25)
for m in ${MODES:-0 1 4 5}; do
  NNM_TC_DBG=$m timeout 300 python tools/quick_perf.py ${1:-2000000x25x4000} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        r=json.loads(l); print('dbg=$m', 'scan_ms=%.1f'%r['scan_ms'], 'items=%d'%r['tc_items'], 'ns_per_item_per_sm=%.1f'%(r['scan_ms']*1e6/r['tc_items']*148), 'rounds', r['boruvka_rounds'], 'amb', r['ambiguous_rows'])"
done
