#!/bin/bash
# next-weights L2 prefetch of the stages AFTER the next launch's ring: A/B over depth
(timeout 600 python -m pytest tests/test_linear_gpu.py -x -q) 2>&1 | tail -1
for pf in 0 1 2 4 -2; do
  if [ "$pf" = "0" ]; then unset ASV_LINEAR_NEXT_PF; else export ASV_LINEAR_NEXT_PF=$pf; fi
  echo "== next_pf=$pf"
  (BATCHES=4,64 timeout 300 python tools/chain_microbench.py) 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['batch'], 'per_gemm', d['per_gemm']['us_per_layer'], 'l2pf', d['per_gemm_l2pf']['us_per_layer'])"
  (timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_npf.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bench_npf.log') if x.startswith('{')][0]; d=json.loads(l); print('bench', round(d['value'],1), round(d['full_decode_step']['hbm_gbps']), round(d['attention_only']['value'],1))"
done
