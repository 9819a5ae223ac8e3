"""Open a composed config through the public API a few times from pinned host
bytes and print each gt_open wall time (GT_TRACE=2 adds the phase timeline).
Diagnostics:  GT_TRACE=2 python tools/open_probe.py c2 [opens]
"""
import sys, time
sys.path.insert(0, ".")
import paper_2106_06889_b200 as gt
from paper_2106_06889_b200.corpus import compose, config_spec
import ctypes as C
import torch
blob, _ = compose(config_spec(sys.argv[1]))
buf = torch.empty(len(blob), dtype=torch.uint8, pin_memory=True)
buf.numpy()[:] = memoryview(blob)
src = (buf.data_ptr(), len(blob))
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 6):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d = gt.DeviceDag(src)
    t1 = time.perf_counter()
    d.close()
    print(f"open {1e3*(t1-t):.3f} ms", file=sys.stderr, flush=True)
