#!/bin/bash
# GQA (C4 shape) vs its MHA control: timing + ncu DRAM bytes of one attention launch and one merge
mkdir -p gpurun_out
for c in C4_13b_gqa8_b32 C4_shape_mha8_b32; do
  timeout 300 python tools/attn_microbench.py --case $c --iters 10
done
for c in C4_13b_gqa8_b32 C4_shape_mha8_b32; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed \
      -k regex:'decode_attn|merge_splits' --launch-skip 40 --launch-count 2 --csv \
      python tools/attn_microbench.py --case $c --iters 2 --warmup 1 > gpurun_out/ncu_gqa_$c.csv 2>&1
  echo "== $c"; grep -E 'decode_attn|merge' gpurun_out/ncu_gqa_$c.csv | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | head -12
done
