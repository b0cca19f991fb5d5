#!/bin/bash
mkdir -p gpurun_out
(BATCH=4 timeout 300 python tools/chain_trace.py; BATCH=64 timeout 300 python tools/chain_trace.py) > gpurun_out/chain_trace.log 2>&1; echo "trace rc=$?"; cat gpurun_out/chain_trace.log
ASV_WATCHDOG=1 timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -5 gpurun_out/ncu_smoke.log
