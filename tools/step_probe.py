#!/usr/bin/env python3
"""The bench step (word count + inverted index through gt_run_many) run a few
times on one config; with GT_TRACE=2 the fused launch prints its phase times
(seeds, every level, word reduce + root words, compaction).  Diagnostics.

    GT_TRACE=2 python tools/step_probe.py c2 --reps 5
"""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    blob, _ = compose(config_spec(a.config, scale=a.scale))
    dag = gt.DeviceDag(blob)
    ids = [gt._abi.TASK_IDS[t] for t in ("wordcount", "invertedindex")]
    for _ in range(a.reps):
        rs = dag.run_many_raw(ids)
        print(f"step device {rs[0][1].device_ms:.4f} ms  d2h {rs[0][1].d2h_ms:.4f} ms", flush=True)
        for r, _ in rs:
            dag.free_raw(r)


if __name__ == "__main__":
    main()
