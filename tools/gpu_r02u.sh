#!/bin/bash
# 1-warp CTAs for the decode attention (ASV_ATTN_VARIANT=1x3) vs the 4-warp default
(ASV_ATTN_VARIANT=1x3 timeout 900 python -m pytest tests/test_attention_gpu.py -x -q) 2>&1 | tail -1
for v in 4x3 1x3; do
  export ASV_ATTN_VARIANT=$v
  echo "== variant $v"
  timeout 300 python tools/attn_warp_timeline.py 2>&1 | grep -E 'C4|C2|launch 5|launch 6'
  timeout 900 python tools/run_configs.py --only c1_7b_b16,c2_7b_1024req,c4_13b_gqa8,c5_zipf_128k 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print(d['config'], d['policy'], round(d['value']['tok_s'],1), round(d['value']['attn_gbps']))"
  (timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_v.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bench_v.log') if x.startswith('{')][0]; d=json.loads(l); print('bench', round(d['value'],1), round(d['full_decode_step']['hbm_gbps']), round(d['attention_only']['value'],1), round(d['roofline']['achieved']))"
done
