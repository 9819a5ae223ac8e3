#!/usr/bin/env python3
"""Top SASS instructions of one kernel in an ncu report by warp-stall samples.

    python tools/ncu_sass_hot.py report.ncu-rep k_kahn [--top 30]
"""
import csv, subprocess, sys, argparse

ap = argparse.ArgumentParser()
ap.add_argument("rep"); ap.add_argument("kernel"); ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "-k", f"regex:{a.kernel}", "--page", "source", "--csv",
                      "--print-source=sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != hdr[0]]
tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
print(f"{len(data)} instructions, {tot} samples")
idx = {id(d): i for i, d in enumerate(data)}
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:a.top]:
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{idx[id(d)]:5d} {100*s/max(tot,1):5.1f}%  {d['Source'].strip()[:70]:70s} ex={d['Instructions Executed']} "
          f"l2sec={d.get('L2 Theoretical Sectors Global','')}")
