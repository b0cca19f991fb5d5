"""Deterministic synthetic traces for BASELINE configs C1-C5 (JSONL, reference
trace format: {"arrival_ms", "prompt_tokens", "output_tokens"} per line,
ingested by prefixsim::ingest_trace, reference workload.hpp:135-210).

Traces are needed because generate_synthetic caps long prompts at 8000 tokens
(workload.hpp:70-72) while the configs call for 16K-128K contexts.  Draws use
splitmix64 (prefixsim::Rng) so the files are reproducible byte for byte.
"""
import json
import math
import os

MASK = (1 << 64) - 1


class Rng:
    def __init__(self, seed):
        self.s = seed & MASK

    def next_u64(self):
        self.s = (self.s + 0x9E3779B97F4A7C15) & MASK
        z = self.s
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform_int(self, lo, hi):
        return lo + self.next_u64() % (hi - lo + 1)

    def next_double(self):
        return (self.next_u64() >> 11) * 2.0 ** -53


def uniform_trace(n, lo, hi, out_lo, out_hi, seed):
    r = Rng(seed)
    return [{"arrival_ms": 0.0, "prompt_tokens": r.uniform_int(lo, hi),
             "output_tokens": r.uniform_int(out_lo, out_hi)} for _ in range(n)]


def zipf_trace(n, unit, kmax, s, out_lo, out_hi, seed):
    """prompt = unit * k with P(k) ~ k^-s over 1..kmax (Zipf lengths unit..unit*kmax)."""
    r = Rng(seed)
    w = [k ** -s for k in range(1, kmax + 1)]
    tot = sum(w)
    cdf, acc = [], 0.0
    for x in w:
        acc += x / tot
        cdf.append(acc)
    out = []
    for _ in range(n):
        u = r.next_double()
        lo, hi = 0, kmax - 1
        while lo < hi:
            mid = (lo + hi) // 2
            if cdf[mid] >= u:
                hi = mid
            else:
                lo = mid + 1
        out.append({"arrival_ms": 0.0, "prompt_tokens": unit * (lo + 1),
                    "output_tokens": r.uniform_int(out_lo, out_hi)})
    return out


def mixed_trace(n, seed):
    """C4: mixed lengths — 70% U[256,2047], 25% U[2048,8191], 5% U[8192,16384]."""
    r = Rng(seed)
    out = []
    for _ in range(n):
        u = r.next_double()
        if u < 0.70:
            p = r.uniform_int(256, 2047)
        elif u < 0.95:
            p = r.uniform_int(2048, 8191)
        else:
            p = r.uniform_int(8192, 16384)
        out.append({"arrival_ms": 0.0, "prompt_tokens": p, "output_tokens": r.uniform_int(60, 68)})
    return out


TRACES = {
    "c1_1024x256-2048.jsonl": lambda: uniform_trace(1024, 256, 2048, 60, 68, 101),
    "c2_1024x1k-16k.jsonl": lambda: uniform_trace(1024, 1024, 16384, 60, 68, 102),
    "c3_256x1k-32k.jsonl": lambda: uniform_trace(256, 1024, 32768, 60, 68, 103),
    "c4_2048xmixed.jsonl": lambda: mixed_trace(2048, 104),
    "c5_1024xzipf128-128k.jsonl": lambda: zipf_trace(1024, 128, 1024, 1.1, 60, 68, 105),
}


def main(dst=None):
    dst = dst or os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs", "traces")
    os.makedirs(dst, exist_ok=True)
    for name, fn in TRACES.items():
        with open(os.path.join(dst, name), "w") as f:
            for rec in fn():
                f.write(json.dumps(rec) + "\n")
    print("wrote", len(TRACES), "traces to", dst)


if __name__ == "__main__":
    main()
