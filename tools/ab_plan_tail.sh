#!/bin/bash
# A/B of the planner's small-item tail (ASV_PLAN_TAIL=<percent of each request's pages>)
mkdir -p gpurun_out
: > gpurun_out/ab_tail.txt
for t in 0 15 25 35; do
  r=$(ASV_PLAN_TAIL=$t timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-step 2>/dev/null | tail -1)
  echo "tail=$t bench $r" >> gpurun_out/ab_tail.txt
  for c in C1_b16_256-2048 C2_step_b4_1k-16k C2_aligned_b13_8k C4_13b_gqa8_b32 mha_b1_128k; do
    echo "tail=$t micro $(ASV_PLAN_TAIL=$t python tools/attn_microbench.py --case $c --iters 10 | tail -1)" >> gpurun_out/ab_tail.txt
  done
done
