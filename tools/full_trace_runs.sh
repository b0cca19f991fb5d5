#!/bin/bash
# Whole BASELINE traces executed on one B200 through the reference CLI face (prefixsim_gpu run):
# every iteration's attention and every KV move executed; the decision logs must be byte-identical
# to the reference's (sha256 in tests/golden/golden.json).
mkdir -p gpurun_out/full_runs
for cfg in c1_7b_b16 c2_7b_1024req c5_zipf_128k; do
  t0=$(date +%s); timeout 1200 paper_2605_23389_b200/prefixsim_gpu run --config configs/$cfg.json \
      --out gpurun_out/full_runs/$cfg --host-pool-mib 4096 > gpurun_out/full_runs/$cfg.stdout 2>&1
  rc=$?; echo "$cfg rc=$rc wall=$(( $(date +%s) - t0 ))s sha256=$(sha256sum gpurun_out/full_runs/$cfg/log.jsonl | cut -c1-64)"
  tail -3 gpurun_out/full_runs/$cfg.stdout
  rm -f gpurun_out/full_runs/$cfg/log.jsonl gpurun_out/full_runs/$cfg/*.csv
done
