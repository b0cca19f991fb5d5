#!/bin/bash
# per-config runs (C1-C5): attention-only, e2e, full step, bubble; + deferred-merge A/B on the attention-only step
mkdir -p gpurun_out
(timeout 2400 python tools/run_configs.py --full --e2e --bubble --out gpurun_out/configs_r02.json) > gpurun_out/configs_r02.log 2>&1; echo "configs rc=$?"; tail -3 gpurun_out/configs_r02.log
(ASV_DEFER_MERGE=0 timeout 1200 python tools/run_configs.py --out gpurun_out/configs_r02_nodefer.json) > gpurun_out/configs_r02_nodefer.log 2>&1; echo "nodefer rc=$?"; tail -3 gpurun_out/configs_r02_nodefer.log
