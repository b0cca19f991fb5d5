#!/bin/bash
# ThreadSanitizer run of the host runtime on a GPU box (writes gpurun_out/tsan_*.txt).
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
python - <<'PY'
import json
g = json.load(open("tests/golden/golden.json"))
json.dump(g["configs"]["smoke"], open("/tmp/tsan_smoke.json", "w"))
json.dump(g["configs"]["short95"], open("/tmp/tsan_short95.json", "w"))
PY
export TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 history_size=4 suppressions=tools/tsan/suppressions.txt"
for mode in "smoke 0" "smoke 1" "short95 0"; do
  set -- $mode
  timeout 900 tools/tsan/build/engine_tsan /tmp/tsan_$1.json 32 $2 8 > gpurun_out/tsan_$1_pair$2.txt 2>&1
  echo "tsan $1 pair=$2 rc=$? warnings=$(grep -c 'WARNING: ThreadSanitizer' gpurun_out/tsan_$1_pair$2.txt)"
  tail -2 gpurun_out/tsan_$1_pair$2.txt
done
