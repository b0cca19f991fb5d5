#!/bin/bash
# push-mode split-K epilogue A/B
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_decode_layer_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -3 gpurun_out/linear_tests.log
for pu in 1 0; do
  export ASV_LINEAR_PUSH=$pu
  echo "== push=$pu"
  BATCH=4 timeout 200 python tools/linear_trace.py | tail -10
  (BATCHES=4,16,64 timeout 600 python tools/chain_microbench.py) 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['batch'], d['per_gemm'])"
  (timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_push$pu.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bench_push$pu.log') if x.startswith('{')][0]; d=json.loads(l); print('bench', d['value'], d['full_decode_step']['hbm_gbps'], d['attention_only']['value'])"
done
