#!/bin/bash
# GQA (C4) planner split-size sweep with the deferred merge
for c in 6 8 10 12; do
  if [ $c = 0 ]; then unset ASV_PLAN_CHUNK; else export ASV_PLAN_CHUNK=$c; fi
  echo "== chunk $c"
  timeout 600 python tools/run_configs.py --only c4_13b_gqa8 --bubble 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d['bubble']; print(d['config'], round(d['value']['tok_s'],1), round(d['value']['attn_gbps']), 'idle', round(b['measured_idle_frac'],3))"
done
