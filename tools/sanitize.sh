#!/bin/bash
# compute-sanitizer passes over the GPU tests (run on the GPU box); summary in gpurun_out/sanitize.txt
mkdir -p gpurun_out
out=gpurun_out/sanitize.txt
: > $out
run() {  # tool, pytest selection
  local log=gpurun_out/san_$1_$(echo "$2" | tr '/ :[]' '_____').log
  timeout 1500 compute-sanitizer --tool $1 --print-limit 20 --target-processes all python -m pytest $2 -x -q > $log 2>&1
  echo "$1 $2 rc=$? $(grep -c '========= .*\(Invalid\|Race\|Hazard\|Error\|error\)' $log) findings; $(grep -E 'passed|failed' $log | tail -1)" >> $out
}
run memcheck "tests/test_attention_gpu.py -k fp16"
run memcheck "tests/test_attention_gpu.py -k config1_shape"
run memcheck "tests/test_kv_copy_gpu.py"
run memcheck "tests/test_engine_gpu.py -k aligned"
run racecheck "tests/test_attention_gpu.py -k fp16_kv_matches"
run synccheck "tests/test_attention_gpu.py -k edge_lengths"
cat $out
