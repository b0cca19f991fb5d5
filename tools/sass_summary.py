#!/usr/bin/env python
"""Per-kernel SASS instruction summary of libasv.so (cuobjdump -sass): which data-movement and
math instructions each kernel really uses (UTMALDG / UBLKCP = TMA, UTCHMMA / UTCBAR / LDTM =
tcgen05 + TMEM, HMMA = mma.sync, FHFMA = packed bf16 FMA, SYNCS = mbarrier), with counts.
Usage: python tools/sass_summary.py [libasv.so] > profiles/sass_rNN.txt"""
import collections
import re
import subprocess
import sys

KEYS = ["UTMALDG", "UTMAPF", "UBLKCP", "UTCHMMA", "UTCBAR", "UTCATOM", "LDTM", "STTM", "HMMA", "LDSM", "MOVM",
        "FHFMA", "FFMA", "HFMA2", "SYNCS", "LDG", "STG", "LDS", "STS", "SHFL", "ATOM", "RED", "BAR", "MEMBAR",
        "FENCE", "NANOSLEEP", "CCTL", "ACQBULK", "ELECT"]


def main():
    so = sys.argv[1] if len(sys.argv) > 1 else "paper_2605_23389_b200/libasv.so"
    out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            op = m.group(1)
            kernels[cur][op] += 1
            kernels[cur]["_total"] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(kernels), capture_output=True, text=True).stdout.split("\n")
    print(f"# SASS instruction summary of {so} (cuobjdump -sass; sm_100a)")
    for (name, cnt), dem in zip(kernels.items(), demangle):
        short = re.sub(r"\(.*", "", dem.replace("(anonymous namespace)::", "")).replace("void ", "")
        keys = ", ".join(f"{k} {cnt[k]}" for k in KEYS if cnt.get(k))
        print(f"{short:60s} total {cnt['_total']:5d} | {keys}")


if __name__ == "__main__":
    main()
