"""Time the REAL reference (the gtadoc package, numba backend) beside the C
restatement the bench's reference arm runs (oracle/gt_oracle.c), on the
same composed corpus and step (word count + inverted index), in THIS
container (the reference does not travel to the GPU box).  Output: one JSON
object (profiles/r2_reference_numba.json) — SURVEY §8(d) CPU-baseline
protocol: one warm call (JIT + caches), then the median of 3 with
time.perf_counter, for workers = 1 and os.cpu_count(); build_dag reported
separately as initialization.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba \\
        python tools/reference_numba_probe.py [--config c2] [--scale 1.0]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
TASKS = ("wordcount", "invertedindex")


def med3(fn):
    fn()  # warm (JIT, caches)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--scale", type=float, default=1.0)
    a = ap.parse_args()
    from paper_2106_06889_b200.corpus import compose, config_spec
    blob, stats = compose(config_spec(a.config, scale=a.scale))
    W = stats["W"]
    out = {"config": a.config, "scale": a.scale, "W": W, "R": stats["R"], "E": stats["E"], "F": stats["F"],
           "host": {"cpu_count": os.cpu_count()}, "step": "+".join(TASKS)}
    # the real reference
    from gtadoc import engine, grammar, tasks
    from gtadoc.dag import build_dag
    t = time.perf_counter()
    g = grammar.deserialize_grammar(blob)
    dag = build_dag(g)
    out["reference_build_dag_s"] = time.perf_counter() - t
    ref = {}
    for w in sorted({1, os.cpu_count() or 1}):
        cfg = engine.TraversalConfig(backend="numba", strategy="auto", workers=w)
        s = med3(lambda: [tasks.run_task(dag, task, cfg) for task in TASKS])
        ref[f"workers={w}"] = {"step_s": s, "words_per_s": W / s}
    out["reference_numba"] = ref
    # the bench's reference arm: the C restatement on all host threads
    from oracle.oracle import OracleDag
    import paper_2106_06889_b200 as gt
    t = time.perf_counter()
    od = OracleDag(blob)
    out["port_open_s"] = time.perf_counter() - t
    s = med3(lambda: [gt.run_compact(od, task, gt.TraversalConfig()) for task in TASKS])
    out["port"] = {"threads": od.workers, "step_s": s, "words_per_s": W / s}
    best = min(v["step_s"] for v in ref.values())
    out["port_speedup_over_reference_numba"] = best / s
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
