#!/usr/bin/env python3
"""Per-kernel device time of gt_open (CUDA events per launch, gt_profile on
the whole process) on a warm open from pinned bytes.  Diagnostics:
    python tools/open_kernels_probe.py c2"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    from paper_2106_06889_b200.device import lib
    blob, _ = compose(config_spec(sys.argv[1]))
    buf = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
    buf.numpy()[:] = memoryview(blob)
    L = lib()
    for _ in range(3):  # warm: module loading, pools
        gt.DeviceDag((buf.data_ptr(), len(blob))).close()
    L.gt_profile(None, 1)
    gt.DeviceDag((buf.data_ptr(), len(blob))).close()
    n = L.gt_profile_report(None, None, 0)
    out = C.create_string_buffer(int(n))
    L.gt_profile_report(None, out, n)
    L.gt_profile(None, 0)
    rows = [ln.split("\t") for ln in out.value.decode().splitlines() if ln]
    rows = sorted(((float(ms), int(k), name) for name, k, ms in rows), reverse=True)
    tot = sum(r[0] for r in rows)
    for ms, k, name in rows:
        print(f"{ms * 1e3:9.1f} us {k:4d}x  {name}")
    print(f"{tot * 1e3:9.1f} us total (kernels with per-launch events; the open also has H2D, syncs and gaps)")


if __name__ == "__main__":
    main()
