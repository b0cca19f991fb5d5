#!/bin/bash
mkdir -p gpurun_out
(BATCHES=4,16,64 timeout 600 python tools/chain_microbench.py) > gpurun_out/chain_micro.log 2>&1; echo "micro rc=$?"; cat gpurun_out/chain_micro.log | tail -4
(BATCH=4 timeout 300 python tools/chain_trace.py) > gpurun_out/chain_trace.log 2>&1; echo "trace rc=$?"; cat gpurun_out/chain_trace.log
(timeout 600 python tools/linear_microbench.py) > gpurun_out/linear_micro.log 2>&1; echo "lin micro rc=$?"; tail -20 gpurun_out/linear_micro.log
