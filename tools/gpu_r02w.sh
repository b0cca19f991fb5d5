#!/bin/bash
# in-situ tuning of the linear schedule constants (full decoder step, C2 bench window)
for cfg in "24 0.9" "20 0.9" "28 0.9" "32 0.9" "24 0.85" "24 0.95" "24 0.9"; do
  set -- $cfg
  export ASV_LINEAR_FLYCAP_MB=$1 ASV_LINEAR_FILL=$2
  (timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_t.log 2>&1
  python -c "import json; l=[x for x in open('gpurun_out/bench_t.log') if x.startswith('{')][0]; d=json.loads(l); print('cap $1 fill $2: bench', round(d['value'],1), round(d['full_decode_step']['hbm_gbps']))"
done
