#!/usr/bin/env python
"""PCIe host<->device bandwidth probe (measurement tool, not product code).

Prints the GPU's NUMA locality and measures pinned H2D / D2H copy bandwidth
with the host buffer placed on each NUMA node (placement by first touch from a
thread pinned to that node's CPUs), for one large copy and for the 256 KiB
layer-slice copies the KV moves use.  Used to explain box-to-box differences
of the e2e line (kv_prefetch.h2d_gbps).
"""
from __future__ import annotations

import glob
import json
import os
import subprocess

import torch


def cpulist(s: str) -> list[int]:
    out = []
    for part in s.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            out.extend(range(int(a), int(b) + 1))
        else:
            out.append(int(part))
    return out


def nodes() -> dict[int, list[int]]:
    res = {}
    for p in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
        n = int(p.rsplit("node", 1)[1])
        with open(os.path.join(p, "cpulist")) as f:
            res[n] = cpulist(f.read())
    return res


def gpu_numa(dev: int) -> tuple[int, str]:
    p = torch.cuda.get_device_properties(dev)
    bus = f"{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    path = f"/sys/bus/pci/devices/{bus.lower()}"
    node, cpus = -1, ""
    try:
        with open(path + "/numa_node") as f:
            node = int(f.read())
        with open(path + "/local_cpulist") as f:
            cpus = f.read().strip()
    except OSError:
        pass
    return node, f"{bus} numa_node={node} local_cpus={cpus}"


def bw(src, dst, chunk: int, reps: int, streams: int) -> float:
    n = src.numel()
    ss = [torch.cuda.Stream() for _ in range(streams)]
    torch.cuda.synchronize()
    beg = torch.cuda.Event(enable_timing=True)
    end = torch.cuda.Event(enable_timing=True)
    beg.record()
    for s in ss:
        s.wait_event(beg)
    k = 0
    for _ in range(reps):
        for off in range(0, n, chunk):
            with torch.cuda.stream(ss[k % streams]):
                dst[off:off + chunk].copy_(src[off:off + chunk], non_blocking=True)
            k += 1
    for s in ss:
        torch.cuda.current_stream().wait_stream(s)
    end.record()
    end.synchronize()
    return reps * n / (beg.elapsed_time(end) * 1e-3) / 1e9


def main():
    dev = 0
    torch.cuda.set_device(dev)
    node, desc = gpu_numa(dev)
    info = {"gpu": desc, "nodes": {k: f"{v[0]}-{v[-1]} ({len(v)})" for k, v in nodes().items()},
            "nproc": os.cpu_count()}
    try:
        info["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True,
                                      timeout=30).stdout
    except Exception as e:  # noqa: BLE001
        info["topo"] = str(e)
    size = 1 << 30
    results = []
    orig = os.sched_getaffinity(0)
    for n, cpus in nodes().items():
        os.sched_setaffinity(0, cpus)
        h = torch.empty(size, dtype=torch.uint8, pin_memory=True)
        h.fill_(1)
        d = torch.empty(size, dtype=torch.uint8, device=dev)
        row = {"host_node": n}
        for name, chunk, streams in (("1GiB", size, 1), ("256KiB", 256 << 10, 1), ("256KiB_2str", 256 << 10, 2),
                                     ("8MiB", 8 << 20, 1)):
            bw(h, d, chunk, 1, streams)
            row[f"h2d_{name}"] = round(bw(h, d, chunk, 3, streams), 2)
            row[f"d2h_{name}"] = round(bw(d, h, chunk, 3, streams), 2)
        results.append(row)
        del h, d
        torch.cuda.empty_cache()
    os.sched_setaffinity(0, orig)
    info["results"] = results
    print(json.dumps(info, indent=1))


if __name__ == "__main__":
    main()
