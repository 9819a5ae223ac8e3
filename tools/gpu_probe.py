#!/usr/bin/env python3
"""Per-config probe on a B200: gt_open phase times, per-task device time and
the top kernels of each task (CUDA-event profile).  Diagnostic only.

    GT_TRACE=1 python tools/gpu_probe.py c2 c3 --tasks wordcount,invertedindex
"""

from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--tasks", default="wordcount,sort,invertedindex,termvector,seqcount,rankedinvertedindex")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--strategy", default="auto", choices=["auto", "topdown", "bottomup"])
    ap.add_argument("--pinned", action="store_true", help="open from a pinned host copy (as bench e2e)")
    ap.add_argument("--top", type=int, default=6, help="kernels listed per task")
    a = ap.parse_args()
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200 import device
    from paper_2106_06889_b200.corpus import compose, config_spec
    for name in a.configs:
        t = time.perf_counter()
        blob, stats = compose(config_spec(name, scale=a.scale))
        print(f"== {name}: composed in {time.perf_counter() - t:.1f}s  "
              f"{json.dumps({k: v for k, v in stats.items() if k != 'spec'})}", flush=True)
        src = blob
        if a.pinned:
            import numpy as np
            import torch
            pin = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
            pin.numpy()[:] = np.frombuffer(blob, dtype=np.uint8)
            src = (pin.data_ptr(), len(blob))
        for rep in range(4):
            # reps 0-2 unprofiled (per-launch events cost host time), rep 3 profiled
            device.profile(rep == 3)
            t = time.perf_counter()
            dag = gt.DeviceDag(src)
            wall = (time.perf_counter() - t) * 1e3
            rp = device.profile_report()
            device.profile(False)
            ktot = sum(ms for _, ms in rp.values())
            print(f"  gt_open rep{rep}: wall {wall:.2f} ms, init_ms {dag.info['init_ms']:.2f}, "
                  f"kernels {ktot:.2f} ms in {sum(n for n, _ in rp.values())} launches", flush=True)
            if rep == 3:
                for k, (n, ms) in sorted(rp.items(), key=lambda kv: -kv[1][1])[:8]:
                    print(f"      {ms:9.3f} ms {n:5d}x  {k}")
                break
            dag.close()
        print(f"  info {json.dumps(dag.info)}", flush=True)
        for task in a.tasks.split(","):
            try:
                # reps unprofiled (the reported device time is their minimum), then
                # one profiled rep for the kernel table
                best = None
                for rep in range(a.reps + 1):
                    dag.profile(rep == a.reps)
                    r, v = dag.run_raw(gt._abi.TASK_IDS[task], 3, gt._abi.STRATEGY_IDS[a.strategy])
                    if rep < a.reps and (best is None or v.device_ms < best[0]):
                        best = (v.device_ms, v.d2h_ms, v.total_ms)
                    dag.free_raw(r)
                dms, d2h, tot = best
                line = (f"  {task:20s} [{gt._abi.STRATEGY_NAMES.get(v.strategy)}] device {dms:9.3f} ms  d2h {d2h:8.3f} ms "
                        f"total {tot:9.3f} ms  n={v.n} groups={v.n_groups} "
                        f"launches={v.kernel_launches} W/s={dag.info['words'] / (dms / 1e3):.3e}")
                print(line, flush=True)
                rp = dag.profile_report()
                dag.profile(False)
                for k, (n, ms) in sorted(rp.items(), key=lambda kv: -kv[1][1])[:a.top]:
                    print(f"      {ms:9.3f} ms {n:5d}x  {k}")
            except Exception as e:  # noqa: BLE001
                dag.profile(False)
                print(f"  {task:20s} FAILED {type(e).__name__}: {e}", flush=True)
        dag.close()


if __name__ == "__main__":
    main()
