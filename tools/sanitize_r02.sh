#!/bin/bash
# compute-sanitizer passes over the round-2 kernels and paths (run on the GPU box)
mkdir -p gpurun_out
out=gpurun_out/sanitize_r02.txt
: > $out
run() {  # tool, pytest selection
  local log=gpurun_out/san_$1_$(echo "$2" | tr '/ :[]' '_____').log
  timeout 1500 compute-sanitizer --tool $1 --print-limit 20 --target-processes all python -m pytest $2 -x -q > $log 2>&1
  echo "$1 $2 rc=$? $(grep -c '========= .*\(Invalid\|Race\|Hazard\|Error\|error\)' $log) findings; $(grep -E 'passed|failed' $log | tail -1)" >> $out
}
run memcheck "tests/test_attention_gpu.py -k deferred"
run racecheck "tests/test_attention_gpu.py -k deferred"
run memcheck "tests/test_linear_gpu.py -k every_schedule"
run memcheck "tests/test_linear_gpu.py -k chain"
run racecheck "tests/test_linear_gpu.py -k chain_decoder"
run synccheck "tests/test_linear_gpu.py -k chain_decoder"
run memcheck "tests/test_engine_content_gpu.py -k single_gpu"
run memcheck "tests/test_decode_layer_gpu.py"
cat $out
