#!/bin/bash
# round 2: chain perf fix check, engine tests (wall clock, whole-C1 page tables), serial / ncu smoke debug, TSan
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_linear_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -2 gpurun_out/linear_tests.log
(timeout 600 python tools/chain_microbench.py) > gpurun_out/chain_micro.log 2>&1; echo "chain micro rc=$?"; tail -6 gpurun_out/chain_micro.log
(timeout 1200 python -m pytest tests/test_engine_gpu.py -x -q) > gpurun_out/engine_tests.log 2>&1; echo "engine tests rc=$?"; tail -3 gpurun_out/engine_tests.log
(ASV_SERIAL=1 ASV_WATCHDOG=1 timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke_serial.log 2>&1; echo "smoke serial rc=$?"; tail -4 gpurun_out/smoke_serial.log
ASV_WATCHDOG=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -12 gpurun_out/ncu_smoke.log
export TSAN_OPTIONS="halt_on_error=0 second_deadlock_stack=1 history_size=4 suppressions=tools/tsan/suppressions.txt"
python - <<'PY'
import json
g = json.load(open("tests/golden/golden.json"))
json.dump(g["configs"]["smoke"], open("/tmp/tsan_smoke.json", "w"))
PY
timeout 600 tools/tsan/build/engine_tsan /tmp/tsan_smoke.json 32 0 8 > gpurun_out/tsan_smoke_pair0.txt 2>&1
echo "tsan smoke rc=$? warnings=$(grep -c 'WARNING: ThreadSanitizer' gpurun_out/tsan_smoke_pair0.txt)"; tail -2 gpurun_out/tsan_smoke_pair0.txt
