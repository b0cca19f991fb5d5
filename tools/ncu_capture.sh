#!/bin/bash
# One gpurun call: ncu evidence for the bench step (run from the repo root on the GPU box).
#   1. launch list of the headline step (cold-cache, serialised: compare SHARES, not absolutes)
#   2. --set full capture of 3 decode-attention launches + 3 merge launches of the same step
#   3. --set full capture of the four linear kernels + rmsnorm of the full decoder step
# Outputs under gpurun_out/ (summarise with tools/ncu_summarize.py).
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-full-step --no-cpu-baseline --steps 3 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'decode_attn|merge_splits' \
    --launch-skip 96 --launch-count 6 -o gpurun_out/prof_bench -f $B > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'linear_kernel|rmsnorm' \
    --launch-skip 200 --launch-count 6 -o gpurun_out/prof_linear -f python tools/full_step_run.py \
    > gpurun_out/ncu_linear.log 2>&1; echo "linear rc=$?"
ls -la gpurun_out
