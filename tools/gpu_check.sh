#!/bin/bash
# One gpurun call: GPU parity tests, smoke, default bench (outputs under gpurun_out/).
mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
(time timeout 1500 python -m pytest tests -m gpu -x -q) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/gpu_tests.log
(time timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/smoke.log
(time timeout 900 python bench.py) > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
