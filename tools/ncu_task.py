#!/usr/bin/env python3
"""Run one config's tasks once each (after a warm-up) for ncu captures.

    ncu ... python tools/ncu_task.py c5 wordcount termvector
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    name, tasks = sys.argv[1], sys.argv[2:]
    scale = 1.0
    if "@" in name:
        name, scale = name.split("@")
        scale = float(scale)
    blob, _ = compose(config_spec(name, scale=scale))
    dag = gt.DeviceDag(blob)
    for t in tasks:
        gt.run_compact(dag, t, gt.TraversalConfig(), 3)
    dag.close()


if __name__ == "__main__":
    main()
