#!/bin/bash
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_linear_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -2 gpurun_out/linear_tests.log
(BATCHES=4,16,64,128 timeout 900 python tools/chain_microbench.py) > gpurun_out/chain_micro.log 2>&1; echo "micro rc=$?"; cat gpurun_out/chain_micro.log
for pf in 0 -1 2 8; do
  if [ "$pf" = "-1" ]; then unset ASV_LINEAR_NEXT_PF; else export ASV_LINEAR_NEXT_PF=$pf; fi
  (timeout 600 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_pf$pf.log 2>&1
  echo "bench pf=$pf rc=$? $(python -c "import json,sys; l=[x for x in open('gpurun_out/bench_pf$pf.log') if x.startswith('{')][0]; d=json.loads(l); print(d['value'], d['full_decode_step']['hbm_gbps'], d['attention_only']['value'])")"
done
unset ASV_LINEAR_NEXT_PF
