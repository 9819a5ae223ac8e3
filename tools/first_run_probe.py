#!/usr/bin/env python3
"""The bench step on FRESH DAGs (what bench.py's e2e times: gt_open from pinned
bytes, then the first word count + inverted index on that DAG, then
gt_close), with the library's own device / D2H / total split per result.
Diagnostics:  python tools/first_run_probe.py c5 [reps]"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    blob, _ = compose(config_spec(sys.argv[1]))
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    buf = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
    buf.numpy()[:] = memoryview(blob)
    ids = [gt._abi.TASK_IDS[t] for t in ("wordcount", "invertedindex")]
    for i in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        d = gt.DeviceDag((buf.data_ptr(), len(blob)))
        t1 = time.perf_counter()
        rs = d.run_many_raw(ids)
        t2 = time.perf_counter()
        parts = [(v.device_ms, v.d2h_ms, v.total_ms, v.kernel_launches, v.d2h_bytes) for _, v in rs]
        for r, _ in rs:
            d.free_raw(r)
        t3 = time.perf_counter()
        d.close()
        t4 = time.perf_counter()
        print(f"open {1e3*(t1-t0):.3f} ms | run_many {1e3*(t2-t1):.3f} ms "
              f"{['dev %.3f d2h %.3f tot %.3f launches %d bytes %d' % p for p in parts]} | free {1e3*(t3-t2):.3f} "
              f"| close {1e3*(t4-t3):.3f} ms", flush=True)


if __name__ == "__main__":
    main()
