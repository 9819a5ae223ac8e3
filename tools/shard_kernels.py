#!/usr/bin/env python3
"""Kernel table of one task on one file-range shard (1 of N) vs the whole
corpus: where a shard's fixed cost goes.  Diagnostics.

    python tools/shard_kernels.py c3 --shards 8 --tasks wordcount,invertedindex
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--tasks", default="wordcount,invertedindex")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    from paper_2106_06889_b200.shard import shard_ranges
    blob, _ = compose(config_spec(a.config))
    dag = gt.DeviceDag(blob)
    ranges = shard_ranges(dag.dag_array("segment_token_counts"), a.shards)
    for label, (lo, hi) in (("whole", (0, 1 << 62)), (f"shard 0/{a.shards}", ranges[0])):
        dag.set_files(lo, hi)
        for task in a.tasks.split(","):
            tid = gt._abi.TASK_IDS[task]
            best = None
            for rep in range(a.reps + 1):
                dag.profile(rep == a.reps)
                r, v = dag.run_raw(tid)
                if rep < a.reps:
                    best = min(best or 1e9, v.device_ms)
                dag.free_raw(r)
            rp = dag.profile_report()
            dag.profile(False)
            print(f"{label:12s} {task:15s} device {best:.3f} ms (profiled rep: {v.device_ms:.3f} ms, "
                  f"{v.kernel_launches} launches)")
            for k, (n, ms) in sorted(rp.items(), key=lambda kv: -kv[1][1])[:10]:
                print(f"      {ms:8.3f} ms {n:4d}x  {k}")


if __name__ == "__main__":
    main()
