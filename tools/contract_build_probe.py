import sys
sys.path.insert(0, ".")
import paper_2106_06889_b200 as gt
from paper_2106_06889_b200.corpus import compose, config_spec
blob, _ = compose(config_spec(sys.argv[1]))
dag = gt.DeviceDag(blob)
ids = [gt._abi.TASK_IDS[t] for t in ("wordcount", "invertedindex")]
for r, _ in dag.run_many_raw(ids): dag.free_raw(r)
dag.profile(True)
for r, _ in dag.run_many_raw(ids): dag.free_raw(r)
rep = dag.profile_report()
dag.profile(False)
tot = 0
for k, (n, ms) in sorted(rep.items(), key=lambda kv: -kv[1][1]):
    tot += ms
    print(f"{ms*1e3:9.1f} us {n:4d}x  {k}")
print("total", tot)
