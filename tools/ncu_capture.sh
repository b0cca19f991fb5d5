#!/bin/bash
# One gpurun call: ncu evidence (run from the repo root on the GPU box).
#   1. launch list of the bench step (full decoder step + attention-only step; cold-cache,
#      serialised: compare SHARES, not absolutes)
#   2. --set full capture of ONE decode-attention launch (+ its merge) of the bench's first timed
#      iteration, with that launch's algorithmic bytes (tools/ncu_bench_launch.py)
#   3. --set full capture of the four linear kernels of the full decoder step
#   4. launch list of __graft_entry__.smoke() (the engine runs in serial mode under ncu)
# Outputs under gpurun_out/ (summarise with tools/ncu_summarize.py).
mkdir -p gpurun_out
B="python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/launches_bench.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'decode_attn|merge_splits' \
    --launch-skip 64 --launch-count 2 -o gpurun_out/prof_bench -f python tools/ncu_bench_launch.py \
    > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'linear_kernel' \
    --launch-skip 200 --launch-count 4 -o gpurun_out/prof_linear -f python tools/full_step_run.py \
    > gpurun_out/ncu_linear.log 2>&1; echo "linear rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -2 gpurun_out/ncu_smoke.log
ls -la gpurun_out
