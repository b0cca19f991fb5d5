#!/bin/bash
# A/B of the plan's pages-per-item (ASV_PLAN_CHUNK) on the attention microbench cases
mkdir -p gpurun_out
for c in 0 8 12 16 24 32; do
  for case in C1_b16_256-2048 C2_step_b4_1k-16k C2_aligned_b13_8k C4_13b_gqa8_b32; do
    r=$(ASV_PLAN_CHUNK=$c python tools/attn_microbench.py --case $case --iters 20 2>&1 | tail -1)
    echo "chunk=$c $r"
  done
done | tee gpurun_out/ab_chunk.txt
