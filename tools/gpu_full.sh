#!/bin/bash
# Full round-end style validation: GPU tests, smoke, smoke under ncu (launch list), default bench.
mkdir -p gpurun_out
(time timeout 2400 python -m pytest tests -m gpu -q) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -4 gpurun_out/gpu_tests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -1 gpurun_out/ncu_smoke.log
(time timeout 900 python bench.py) > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; head -c 400 gpurun_out/bench.log
