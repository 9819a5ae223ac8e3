#!/usr/bin/env python3
"""Summarise a tools/profile_round.sh capture into markdown (profiles/).

    python tools/summarize_profiles.py gpurun_out/prof_r1a > profiles/r1_summary.md
"""

from __future__ import annotations

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path


def rows_of(path: Path):
    rows = list(csv.reader(path.open()))
    i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
    return rows[i], rows[i + 1:]


def short(name: str) -> str:
    n = name.replace("void ", "").replace("gt::", "").replace("<unnamed>::", "")
    return n.split("(")[0][:70]


def per_launch_metrics(path: Path):
    hdr, data = rows_of(path)
    by = defaultdict(dict)
    names = {}
    for r in data:
        d = dict(zip(hdr, r))
        names[d["ID"]] = short(d["Kernel Name"])
        try:
            v = float(d["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        u = d["Metric Unit"]
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ns": 1e-9, "us": 1e-6,
                 "ms": 1e-3}.get(u, 1.0)
        by[d["ID"]][d["Metric Name"]] = v * scale
    return names, by


def main():
    cap = Path(sys.argv[1])
    out = []
    bench = json.loads((cap / "bench.json").read_text().strip().splitlines()[-1])
    out.append(f"# Profile summary — `{cap.name}`\n")
    out.append("Source: `tools/profile_round.sh` under gpurun on one B200; raw files in "
               f"`gpurun_out/{cap.name}/` (launch list, metrics, `--set full` report).  "
               "ncu times are cold-cache and serialised: compare shares, not absolutes.\n")
    out.append("## Bench line (no profiler)\n")
    keep = {k: bench[k] for k in ("value", "unit", "ms_per_step", "n_gpus", "dtype")}
    out.append("```\n" + json.dumps(keep) + "\n```")
    out.append(f"* e2e: `{json.dumps(bench['e2e'])}`")
    out.append(f"* roofline: `{json.dumps(bench['roofline'])}`")
    out.append(f"* cpu_baseline: `{json.dumps(bench['cpu_baseline'])}`")
    out.append(f"* clocks: `{json.dumps(bench['clocks'])}`\n")

    # launch list: the last bench step = launches after the last gt_open of the
    # timed steps; report kernel shares over the whole capture's task kernels
    hdr, data = rows_of(cap / "launches.csv")
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in data:
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", "")) * (1e-3 if d["Metric Unit"] == "ns" else 1.0)
        k = short(d["Kernel Name"])
        tot[k] += v
        cnt[k] += 1
    s = sum(tot.values())
    out.append("## Launch list (whole `bench.py --steps 2 --warmup 3` run, incl. gt_open)\n")
    out.append("| kernel | launches | total µs | share |")
    out.append("|---|---:|---:|---:|")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:20]:
        out.append(f"| `{k}` | {cnt[k]} | {v:.1f} | {v / s:.1%} |")

    names, by = per_launch_metrics(cap / "metrics.csv")
    agg = defaultdict(lambda: defaultdict(list))
    for i, m in by.items():
        for k, v in m.items():
            agg[names[i]][k].append(v)
    out.append("\n## Per-launch DRAM traffic of the step kernels (averages over launches)\n")
    out.append("| kernel | launches | µs | DRAM read MB | DRAM write MB | DRAM % of peak | L2 red sectors | L2 atom sectors |")
    out.append("|---|---:|---:|---:|---:|---:|---:|---:|")
    for k, m in sorted(agg.items(), key=lambda kv: -sum(kv[1]["gpu__time_duration.sum"])):
        n = len(m["gpu__time_duration.sum"])
        a = lambda key: sum(m[key]) / max(1, len(m[key]))  # noqa: E731
        out.append(f"| `{k}` | {n} | {a('gpu__time_duration.sum') * 1e6:.1f} | "
                   f"{a('dram__bytes_read.sum') / 1e6:.2f} | {a('dram__bytes_write.sum') / 1e6:.2f} | "
                   f"{a('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                   f"{a('lts__t_sectors_op_red.sum'):.0f} | {a('lts__t_sectors_op_atom.sum'):.0f} |")

    rep = cap / "full.ncu-rep"
    if rep.exists():
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True,
                             text=True).stdout.splitlines()
        rr = list(csv.reader(raw))
        if len(rr) > 2:
            h = rr[0]
            want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
                    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
                    "sm__warps_active.avg.pct_of_peak_sustained_active",
                    "launch__registers_per_thread", "launch__occupancy_limit_registers",
                    "launch__grid_size", "smsp__average_warp_latency_issue_stalled_long_scoreboard",
                    "smsp__warp_issue_stalled_barrier_per_warp_active.pct",
                    "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct",
                    "smsp__warp_issue_stalled_membar_per_warp_active.pct",
                    "smsp__warp_issue_stalled_lg_throttle_per_warp_active.pct"]
            out.append(f"\n## `ncu --set full` of the dominant kernel ({short(rr[2][h.index('Kernel Name')])})\n")
            out.append("| metric | " + " | ".join(f"launch {j}" for j in range(len(rr) - 2)) + " | unit |")
            out.append("|---|" + "---:|" * (len(rr) - 2) + "---|")
            for w in want:
                if w in h:
                    c = h.index(w)
                    out.append(f"| `{w}` | " + " | ".join(r[c] for r in rr[2:]) + f" | {rr[1][c]} |")
    print("\n".join(out))


if __name__ == "__main__":
    main()
