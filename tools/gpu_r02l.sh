#!/bin/bash
# GQA (C4) with the deferred merge: planner small-item tail sweep
for t in 0 10 25 35; do
  echo "== tail $t"
  ASV_PLAN_TAIL=$t timeout 600 python tools/run_configs.py --only c4_13b_gqa8,c1_7b_b16 --bubble 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d['bubble']; print(d['config'], round(d['value']['tok_s'],1), round(d['value']['attn_gbps']), 'idle', round(b['measured_idle_frac'],3))"
done
