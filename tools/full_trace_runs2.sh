#!/bin/bash
# More whole traces on one B200 (see tools/full_trace_runs.sh): C3 with the pair's data path on one
# device (admits/evicts are real device copies), C5 under FCFS (swap-in/out over PCIe)
mkdir -p gpurun_out/full_runs
run() {  # name, extra flags
  local name=$1; shift
  t0=$(date +%s); timeout 1200 paper_2605_23389_b200/prefixsim_gpu run --out gpurun_out/full_runs/$name --host-pool-mib 4096 "$@" \
      > gpurun_out/full_runs/$name.stdout 2>&1
  rc=$?; echo "$name rc=$rc wall=$(( $(date +%s) - t0 ))s sha256=$(sha256sum gpurun_out/full_runs/$name/log.jsonl | cut -c1-64)"
  tail -3 gpurun_out/full_runs/$name.stdout
  rm -f gpurun_out/full_runs/$name/log.jsonl gpurun_out/full_runs/$name/*.csv
}
run c3_pair_32k --config configs/c3_pair_32k.json --pair-mode
run c5_zipf_128k_fcfs --config configs/c5_zipf_128k.json --policy fcfs
