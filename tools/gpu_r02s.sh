#!/bin/bash
# whole traces executed on one B200 with the round-2 orchestrator / executor; logs vs golden sha256
bash tools/full_trace_runs.sh 2>&1 | tee gpurun_out/full_runs_a.txt
bash tools/full_trace_runs2.sh 2>&1 | tee gpurun_out/full_runs_b.txt
python - <<'PY'
import json, re
g = json.load(open("tests/golden/golden.json"))["logs"]
want = {"c1_7b_b16": "c1_7b_b16:aligned", "c2_7b_1024req": "c2_7b_1024req:aligned", "c5_zipf_128k": "c5_zipf_128k:aligned",
        "c3_pair_32k": "c3_pair_32k:aligned", "c5_zipf_128k_fcfs": "c5_zipf_128k:fcfs"}
for f in ("gpurun_out/full_runs_a.txt", "gpurun_out/full_runs_b.txt"):
    for line in open(f):
        m = re.match(r"(\S+) rc=(\d+) wall=(\d+)s sha256=([0-9a-f]+)", line)
        if m:
            name, rc, wall, sha = m.groups()
            ok = sha == g[want[name]]["sha256"]
            print(f"{name}: rc={rc} wall={wall}s log sha256 {'== golden' if ok else '!= golden ' + sha[:16]}")
PY
