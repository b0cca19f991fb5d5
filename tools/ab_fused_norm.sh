#!/bin/bash
# A/B of the fused RMSNorm in the full decode step (ASV_UNFUSED_NORM=1: standalone norm kernels)
mkdir -p gpurun_out
: > gpurun_out/ab_fnorm.txt
for rep in 1 2; do for v in fused unfused; do for cfg in c2_7b_1024req c1_7b_b16 c5_zipf_128k; do
  if [ $v = unfused ]; then export ASV_UNFUSED_NORM=1; else unset ASV_UNFUSED_NORM; fi
  echo "$v $cfg $(STEPS=40 CONFIG=$cfg timeout 300 python tools/full_step_run.py | tail -1)" >> gpurun_out/ab_fnorm.txt
done; done; done
