import sys, time
sys.path.insert(0, '.')
import paper_2106_06889_b200 as gt
from paper_2106_06889_b200.corpus import compose, config_spec
blob, _ = compose(config_spec(sys.argv[1]))
dag = gt.DeviceDag(blob)
for task in sys.argv[2].split(','):
    tid = gt._abi.TASK_IDS[task]
    for rep in range(4):
        t = time.perf_counter()
        r, v = dag.run_raw(tid)
        w = (time.perf_counter() - t) * 1e3
        print(f"{task} rep{rep}: device {v.device_ms:.3f} d2h {v.d2h_ms:.3f} ms ({v.d2h_bytes/1e6:.1f} MB) wall {w:.1f} ms", flush=True)
        dag.free_raw(r)
