#!/bin/bash
# epilogue staging A/B: linear tests, timeline, per-GEMM stack, bench full step
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_linear_gpu.py tests/test_decode_layer_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -2 gpurun_out/linear_tests.log
for ns in 0 1; do
  if [ $ns = 1 ]; then export ASV_LINEAR_NO_STAGE=1; else unset ASV_LINEAR_NO_STAGE; fi
  echo "== no_stage=$ns"
  BATCH=4 timeout 200 python tools/linear_trace.py | tail -3
  BATCH=64 timeout 200 python tools/linear_trace.py | tail -2
  (BATCHES=4,16,64 timeout 600 python tools/chain_microbench.py) 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['batch'], d['per_gemm'])"
  (timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_ns$ns.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bench_ns$ns.log') if x.startswith('{')][0]; d=json.loads(l); print('bench', d['value'], d['full_decode_step']['hbm_gbps'], d['attention_only']['value'])"
done
