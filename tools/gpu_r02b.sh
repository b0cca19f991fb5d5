#!/bin/bash
# round 2: chain-kernel validation + A/B, smoke, bench, smoke under ncu, TSan (outputs under gpurun_out/)
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_linear_gpu.py -x -q) > gpurun_out/linear_tests.log 2>&1; echo "linear tests rc=$?"; tail -4 gpurun_out/linear_tests.log
(timeout 600 python tools/chain_microbench.py) > gpurun_out/chain_micro.log 2>&1; echo "chain micro rc=$?"; cat gpurun_out/chain_micro.log | tail -8
(timeout 300 python -c "import __graft_entry__ as g; g.smoke()") > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke.log
(timeout 900 python bench.py --no-cpu-baseline) > gpurun_out/bench_chain.log 2>&1; echo "bench chain rc=$?"; tail -c 1500 gpurun_out/bench_chain.log
(ASV_LINEAR_CHAIN=0 timeout 900 python bench.py --no-cpu-baseline --no-e2e) > gpurun_out/bench_nochain.log 2>&1; echo "bench nochain rc=$?"; head -c 600 gpurun_out/bench_nochain.log
(timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_decode_layer_gpu.py -x -q) > gpurun_out/engine_tests.log 2>&1; echo "engine tests rc=$?"; tail -3 gpurun_out/engine_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv \
    --log-file gpurun_out/launches_smoke.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/ncu_smoke.log 2>&1; echo "smoke under ncu rc=$?"; tail -3 gpurun_out/ncu_smoke.log
bash tools/tsan/run.sh
