#!/bin/bash
# gpurun helper: run the given pytest selection (arg 1, may be empty) then bench.py with the remaining args.
mkdir -p gpurun_out
sel="$1"; shift
if [ -n "$sel" ]; then (timeout 1200 python -m pytest $sel -x -q) > gpurun_out/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/tests.log; fi
if [ "$1" != "--no-bench" ]; then (time timeout 900 python bench.py "$@") > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 4000 gpurun_out/bench.log; fi
