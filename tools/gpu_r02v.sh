#!/bin/bash
# the reference's own smoke / short95 configs under aligned / fcfs / disagg-fcfs, executed on the B200
# with the round-2 engine; log sha256 vs the golden digests
bash tools/full_trace_runs_reference_configs.sh 2>&1 | tee gpurun_out/refcfg_runs.txt
python - <<'PY'
import json, re
g = json.load(open("tests/golden/golden.json"))["logs"]
for line in open("gpurun_out/refcfg_runs.txt"):
    m = re.match(r"(\S+)_(aligned|fcfs|disagg-fcfs) rc=(\d+) wall=(\d+)s sha256=([0-9a-f]+)", line)
    if m:
        cfg, pol, rc, wall, sha = m.groups()
        ok = sha == g[f"{cfg}:{pol}"]["sha256"]
        print(f"{cfg}:{pol}: rc={rc} wall={wall}s log sha256 {'== golden' if ok else '!= golden ' + sha[:16]}")
PY
