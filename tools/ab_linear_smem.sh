#!/bin/bash
# A/B of the linear kernels' TMA ring budget (ASV_LINEAR_SMEM_KB) on the full decode step
mkdir -p gpurun_out
: > gpurun_out/ab_lsmem.txt
for rep in 1 2; do
for kb in 100 80 72 64 48; do
  for cfg in c2_7b_1024req c1_7b_b16; do
    echo "kb=$kb cfg=$cfg $(ASV_LINEAR_SMEM_KB=$kb STEPS=40 CONFIG=$cfg timeout 300 python tools/full_step_run.py 2>&1 | tail -1)" >> gpurun_out/ab_lsmem.txt
  done
done
done
