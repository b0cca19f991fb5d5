#!/bin/bash
mkdir -p gpurun_out
(ASV_LINEAR_PLAN_LOG=1 timeout 300 python -m pytest tests/test_linear_gpu.py -x -q -s -k chain 2>&1 | grep -v "^  L") > gpurun_out/chain_tests.log 2>&1; echo "chain tests rc=$?"; tail -15 gpurun_out/chain_tests.log
(BATCHES=4,16,64 timeout 300 python tools/chain_microbench.py) > gpurun_out/chain_micro.log 2>&1; echo "micro rc=$?"; tail -5 gpurun_out/chain_micro.log
(BATCH=4 timeout 120 python tools/chain_trace.py) > gpurun_out/chain_trace.log 2>&1; echo "trace rc=$?"; cat gpurun_out/chain_trace.log
