#!/bin/bash
(timeout 300 python -m pytest tests/test_linear_gpu.py -x -q -k chain) 2>&1 | tail -1
for ns in 2 4; do
  echo "== slots $ns"
  (ASV_CHAIN_SLOTS=$ns BATCHES=4,64 timeout 300 python tools/chain_microbench.py) 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['batch'], d['per_gemm']['us_per_layer'], d['chain']['us_per_layer'])"
  ASV_CHAIN_SLOTS=$ns BATCH=4 timeout 120 python tools/chain_trace.py
done
