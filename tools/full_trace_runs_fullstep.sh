#!/bin/bash
# Whole traces with the full decoder layer stack per iteration (RMSNorm, QKV+RoPE, attention + KV append,
# O + residual, RMSNorm, gate/up SiLU, down + residual; tcgen05 GEMMs) and every KV move executed.
mkdir -p gpurun_out/full_runs
for cfg in c1_7b_b16 c2_7b_1024req; do
  t0=$(date +%s); timeout 1500 paper_2605_23389_b200/prefixsim_gpu run --config configs/$cfg.json --full-step \
      --out gpurun_out/full_runs/${cfg}_full --host-pool-mib 4096 > gpurun_out/full_runs/${cfg}_full.stdout 2>&1
  rc=$?; echo "${cfg}_full rc=$rc wall=$(( $(date +%s) - t0 ))s sha256=$(sha256sum gpurun_out/full_runs/${cfg}_full/log.jsonl | cut -c1-64)"
  tail -3 gpurun_out/full_runs/${cfg}_full.stdout
  rm -f gpurun_out/full_runs/${cfg}_full/log.jsonl gpurun_out/full_runs/${cfg}_full/*.csv
done
