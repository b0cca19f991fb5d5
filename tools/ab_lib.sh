#!/bin/bash
# A/B of two builds of libasv.so (ASV_LIB_PATH) on the attention microbench + bench step.
# usage: tools/ab_lib.sh <base .so> "<cases>"
mkdir -p gpurun_out
base=$1; cases=${2:-"C1_b16_256-2048 C2_step_b4_1k-16k C4_13b_gqa8_b32 gqa_7b_b64"}
: > gpurun_out/ab_lib.txt
for rep in 1 2; do
  for lib in "$base" paper_2605_23389_b200/libasv.so; do
    tag=$(basename $lib)
    for c in $cases; do
      echo "$tag micro $(ASV_LIB_PATH=$lib python tools/attn_microbench.py --case $c --iters 10 | tail -1)" >> gpurun_out/ab_lib.txt
    done
    echo "$tag bench $(ASV_LIB_PATH=$lib timeout 600 python bench.py --no-e2e --no-cpu-baseline --no-full-step 2>/dev/null | tail -1)" >> gpurun_out/ab_lib.txt
  done
done
