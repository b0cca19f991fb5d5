#!/bin/bash
# ring size / co-residency sweep of the per-GEMM linear stack (timeline + stack us/layer)
mkdir -p gpurun_out
(timeout 600 python -m pytest tests/test_linear_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -1 gpurun_out/linear_tests.log
for kb in 100 72 64 56; do
  export ASV_LINEAR_SMEM_KB=$kb
  echo "== smem_kb=$kb"
  BATCH=4 timeout 200 python tools/linear_trace.py | tail -10
  (BATCHES=4,16,64 timeout 600 python tools/chain_microbench.py) 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print(d['batch'], d['per_gemm'])"
done
