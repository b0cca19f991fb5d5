#!/bin/bash
# round-2 final validation: GPU suite, smoke, smoke under ncu, default bench, reference arm
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_info.txt 2>&1
(time timeout 2400 python -m pytest tests -m gpu -q) > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -6 gpurun_out/gpu_tests.log
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
(time timeout 900 python bench.py) > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; grep '^{' gpurun_out/bench.log | head -c 600; echo; tail -4 gpurun_out/bench.log
(time timeout 900 python bench.py --impl reference) > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?"; grep '^{' gpurun_out/bench_ref.log | head -c 600; echo; tail -4 gpurun_out/bench_ref.log
