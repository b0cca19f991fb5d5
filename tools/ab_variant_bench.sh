#!/bin/bash
# A/B of attention kernel variants (ASV_ATTN_VARIANT=<warps>x<stages>) on the headline bench step + microbench shapes
mkdir -p gpurun_out
for rep in 1 2; do
for v in 4x3 4x2; do
  r=$(ASV_ATTN_VARIANT=$v timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-step 2>/dev/null | tail -1)
  echo "$v $r"
done
done > gpurun_out/ab_variant_bench.txt
: > gpurun_out/ab_variant.txt
for v in 4x3 4x2; do for c in C1_b16_256-2048 C2_step_b4_1k-16k C2_aligned_b13_8k C2_b64_1k-16k C4_13b_gqa8_b32 gqa_7b_b64 mha_b1_128k; do
  echo "$v $(ASV_ATTN_VARIANT=$v python tools/attn_microbench.py --case $c --iters 10 | tail -1)"; done; done >> gpurun_out/ab_variant.txt
