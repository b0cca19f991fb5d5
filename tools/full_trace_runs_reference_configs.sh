#!/bin/bash
# The reference's own configs (proj/configs/smoke.json, short95.json; copies in tests/golden/golden.json)
# executed on one B200 through prefixsim_gpu run, under the three policies: every iteration's attention
# and every KV move executed; the logs must equal the reference's (sha256 in golden.json).
mkdir -p gpurun_out/full_runs
python - <<'PY'
import json
g = json.load(open("tests/golden/golden.json"))
for name in ("smoke", "short95"):
    json.dump(g["configs"][name], open(f"gpurun_out/full_runs/{name}.json", "w"))
PY
for name in smoke short95; do for pol in aligned fcfs disagg-fcfs; do
  out=gpurun_out/full_runs/${name}_${pol}
  t0=$(date +%s); timeout 1500 paper_2605_23389_b200/prefixsim_gpu run --config gpurun_out/full_runs/$name.json \
      --policy $pol --out $out --host-pool-mib 4096 > $out.stdout 2>&1
  rc=$?
  got=$(sha256sum $out/log.jsonl | cut -c1-64)
  want=$(python -c "import json; print(json.load(open('tests/golden/golden.json'))['logs']['$name:$pol']['sha256'])")
  echo "$name:$pol rc=$rc wall=$(( $(date +%s) - t0 ))s match=$([ "$got" = "$want" ] && echo yes || echo NO)"
  tail -2 $out.stdout | head -1
  rm -f $out/log.jsonl $out/*.csv
done; done
