"""Summarise ncu captures into profiles/ (committed evidence).

usage: python tools/ncu_summarize.py --launches gpurun_out/launches_bench.csv \
          --full gpurun_out/prof_bench.ncu-rep --tag r01 [--bench-json profiles/bench_r01.json]
Writes profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/ncu_<tag>_{launches,full}.txt.
"""
import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__cycles_elapsed.avg.per_second",
        "launch__shared_mem_per_block_dynamic"]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return float(v.replace(",", "")) * scale


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ik, im, iu, iv = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) > iv and r[im] == "gpu__time_duration.sum":
            ns = float(r[iv].replace(",", "")) * (1e3 if r[iu] == "us" else 1.0)
            name = r[ik].split("(")[0]
            agg[name][0] += 1
            agg[name][1] += ns
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": n, "total_us": t / 1e3, "share": t / tot}
            for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            if w in hdr:
                d[w] = vals[hdr.index(w)] + " " + units[hdr.index(w)]
        d["dram_bytes"] = to_bytes(vals[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")]) + \
            to_bytes(vals[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--alg-bytes-per-launch", type=float, default=None)
    ap.add_argument("--alg-json", default=None, help="gpurun_out/ncu_launch_alg.json of tools/ncu_bench_launch.py")
    a = ap.parse_args()
    alg_src = None
    if a.alg_json:
        rec = json.load(open(a.alg_json))
        a.alg_bytes_per_launch = rec["alg_bytes_per_launch"]
        alg_src = (f"ncu --set full of one decode_attn launch of tools/ncu_bench_launch.py (C2 iteration "
                   f"{rec['iteration']}, batch {rec['batch']}, {rec['tokens']} tokens; tag {a.tag})")
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    summary_path = os.path.join(prof, "ncu_summary.json")
    summary = json.load(open(summary_path)) if os.path.exists(summary_path) else {}
    if a.launches:
        ls = launches(a.launches)
        summary["launch_list"] = {"tag": a.tag, "source": os.path.basename(a.launches),
                                  "note": "ncu --metrics gpu__time_duration.sum --clock-control none "
                                          "(cold-cache, serialised: compare shares)", "kernels": ls}
        with open(os.path.join(prof, f"ncu_{a.tag}_launches.txt"), "w") as f:
            for k in ls:
                f.write(f"{k['launches']:6d} launches {k['total_us']:12.1f} us {100*k['share']:6.1f}%  {k['kernel']}\n")
    if a.full:
        fl = full(a.full)
        main_k = [k for k in fl if "decode_attn" in k["kernel"]]
        per = sum(k["dram_bytes"] for k in main_k) / max(1, len(main_k))
        summary["bench_kernel"] = {"tag": a.tag, "kernel": main_k[0]["kernel"] if main_k else None,
                                   "captures": fl, "dram_bytes_per_launch": per,
                                   "alg_bytes_per_launch": a.alg_bytes_per_launch,
                                   "source": alg_src,
                                   "note": "ncu --set full --clock-control none; one capture per launch"}
        with open(os.path.join(prof, f"ncu_{a.tag}_full.txt"), "w") as f:
            for k in fl:
                f.write(json.dumps(k) + "\n")
    json.dump(summary, open(summary_path, "w"), indent=1)
    print("wrote", summary_path)


if __name__ == "__main__":
    main()
