#!/bin/bash
# planner tail sweep (MHA configs) with the deferred merge
for t in 25 35 50; do
  echo "== tail $t"
  ASV_PLAN_TAIL=$t timeout 900 python tools/run_configs.py --only c1_7b_b16,c2_7b_1024req,c5_zipf_128k --bubble 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); b=d['bubble']; print(d['config'], d['policy'], round(d['value']['tok_s'],1), round(d['value']['attn_gbps']), 'idle', round(b['measured_idle_frac'],3))"
done
for c in 8 12 16; do
  echo "== chunk $c"
  ASV_PLAN_CHUNK=$c timeout 900 python tools/run_configs.py --only c1_7b_b16,c2_7b_1024req 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['policy'], round(d['value']['tok_s'],1), round(d['value']['attn_gbps']))"
done
