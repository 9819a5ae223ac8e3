#!/usr/bin/env python3
"""Per-shard timing of the file-range sharding on ONE GPU: the
device time of each task over the whole corpus vs over 1/N of the files
(token-balanced ranges, shard.shard_ranges).  With the DAG replicated and no
data-path collective for per-file tasks, N GPUs take max over shards of the
shard time (+ the gather), so whole / max-shard bounds the strong scaling.
Diagnostic only.

    python tools/shard_probe.py c3 --shards 8 --tasks invertedindex,termvector
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--tasks", default="invertedindex,termvector")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    from paper_2106_06889_b200.shard import shard_ranges
    blob, _ = compose(config_spec(a.config, scale=a.scale))
    dag = gt.DeviceDag(blob)
    toks = dag.dag_array("segment_token_counts")
    ranges = shard_ranges(toks, a.shards)
    out = {"config": a.config, "shards": a.shards, "files": int(dag.info["num_files"]), "tasks": {}}
    for task in a.tasks.split(","):
        tid = gt._abi.TASK_IDS[task]

        def best(lo, hi):
            dag.set_files(lo, hi)
            ms = []
            for _ in range(a.reps):
                r, v = dag.run_raw(tid)
                ms.append(v.device_ms)
                dag.free_raw(r)
            return min(ms)

        whole = best(0, 1 << 62)
        per = [best(lo, hi) for lo, hi in ranges]
        out["tasks"][task] = {"whole_ms": whole, "shard_ms": per, "max_shard_ms": max(per),
                              "projected_speedup": whole / max(per)}
    dag.set_files(0, 1 << 62)
    dag.close()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
