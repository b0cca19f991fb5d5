#!/bin/bash
# round 2 re-entry: full GPU suite, smoke, smoke under ncu, bench (deferred merge default) + A/B without it
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
(time timeout 2400 python -m pytest tests -m gpu -q -x) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_tests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
(time timeout 900 python bench.py) > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | head -c 700; echo
(ASV_DEFER_MERGE=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_nodefer.log 2>&1; echo "bench nodefer rc=$?"; grep '^{' gpurun_out/bench_nodefer.log | head -c 400; echo
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -3 gpurun_out/ncu_smoke.log
