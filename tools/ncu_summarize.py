#!/usr/bin/env python3
"""Summarise ncu outputs into profiles/ text: per-kernel launch shares from a
`--metrics gpu__time_duration.sum --csv` launch list, and key metrics from a
`--set full` report (ncu -i ... --page details/raw)."""
from __future__ import annotations

import collections
import csv
import subprocess
import sys


def launch_list(path: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
        agg[r[ki].split("(")[0]].append(v)
        if "k_finish" in r[ki]:  # the end of the first run (the bench's later passes add timing / invariant kernels)
            break
    tot = sum(sum(v) for v in agg.values())
    out = [f"# launch list {path}: the first run = {sum(len(v) for v in agg.values())} launches, {tot / 1e3:.3f} ms "
           "(serialised, cold)"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k:40s} n={len(v):5d} sum={sum(v) / 1e3:9.3f} ms avg={sum(v) / len(v):9.2f} us share={sum(v) / tot:.3f}")
    return "\n".join(out)


def full_report(path: str) -> str:
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    h = rows[0]
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
            "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread", "L2 Hit Rate", "L1/TEX Hit Rate",
            "Warp Cycles Per Issued Instruction", "Executed Instructions", "Dynamic Shared Memory Per Block"]
    out = [f"# ncu --set full {path}"]
    for row in rows[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want:
            out.append(f"{d['Kernel Name'].split('(')[0]:14s} id={d['ID']:3s} {d['Metric Name']:36s} {d['Metric Value']} {d['Metric Unit']}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h = rows[0]
    for row in rows[2:]:
        d = dict(zip(h, row))
        vals = []
        for k, v in d.items():
            if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    vals.append((float(v.replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        t = sum(v for v, _ in vals) or 1
        name = d["Kernel Name"].split("(")[0]
        out.append(f"{name:14s} stalls: " + " ".join(f"{k}={v / t:.2f}" for v, k in sorted(vals, reverse=True)[:6]))
        for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
                  "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "gpu__time_duration.sum"):
            if k in d:
                out.append(f"{name:14s} {k} = {d[k]} {rows[1][h.index(k)] if k in h else ''}")
    return "\n".join(out)


def traffic_json(path: str, config: int, out: str) -> dict:
    """profiles/ncu_traffic.json: dram__bytes_read.sum + dram__bytes_write.sum
    per launch of each wave kernel (mean over the captured launches), tagged
    with the hash of the kernel sources bench.py compares before using it."""
    import json
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import kernel_src_sha
    acc = collections.defaultdict(list)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for one in path.split(","):  # several reports: e.g. the wave kernels and the per-window walk
        raw = subprocess.run(["ncu", "-i", one, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h = rows[0]
        unit = rows[1]
        for row in rows[2:]:
            d = dict(zip(h, row))
            name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("eg::", "").split("<")[0]
            b = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                b += float(d[k].replace(",", "")) * scale.get(unit[h.index(k)], 1)
            acc[name].append(b)
    res = {"kernel_src_sha": kernel_src_sha(), "config": config, "source": ",".join(os.path.basename(x) for x in path.split(",")),
           "per_launch_bytes": {k: round(sum(v) / len(v)) for k, v in acc.items()}}
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    return res


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--traffic":
        print(traffic_json(sys.argv[2], int(sys.argv[3]), sys.argv[4]))
        sys.exit(0)
    for p in sys.argv[1:]:
        print(full_report(p) if p.endswith(".ncu-rep") else launch_list(p))
        print()
