"""TEST INFRASTRUCTURE — run the CPU oracle (oracle/gt_oracle.c) in a child
process under an address-space limit, for the full-size parity tests whose
oracle needs tens of GB of host RAM (the reference's dense R x F segment
counts, dag.py:75-86, and token-sized gram tables, sequence.py:319-321).
A limit hit fails the oracle with a ResourceError in the child instead of
taking the host down; the parent never maps the oracle's memory.

    python tests/oracle_worker.py <blob.gtdc> <out.npz> <task[,task...]> <seq_len> <limit_gb>
"""

from __future__ import annotations

import resource
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

FIELDS = ["group_off", "group_id", "group_key", "group_gram", "id", "key", "gram", "count"]


def main():
    blob_path, out_path, tasks, l, limit_gb = sys.argv[1:6]
    lim = int(float(limit_gb) * (1 << 30))
    resource.setrlimit(resource.RLIMIT_AS, (lim, lim))
    import numpy as np
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    ref = OracleDag(Path(blob_path).read_bytes())
    arrs = {}
    for task in tasks.split(","):
        c = gt.run_compact(ref, task, gt.TraversalConfig(), int(l))
        arrs[f"{task}.meta"] = np.asarray([c.n, c.n_groups, c.wbits], dtype=np.int64)
        for f in FIELDS:
            v = getattr(c, f)
            if v is not None:
                arrs[f"{task}.{f}"] = v
    np.savez(out_path, **arrs)


def run(blob: bytes, tasks, seq_len: int, limit_gb: float, tmp: Path):
    """Parent side: the oracle's compact results per task as SimpleNamespaces
    (the fields assert_same compares)."""
    import subprocess
    from types import SimpleNamespace

    import numpy as np
    bp, op = tmp / "in.gtdc", tmp / "out.npz"
    bp.write_bytes(blob)
    r = subprocess.run([sys.executable, __file__, str(bp), str(op), ",".join(tasks), str(seq_len), str(limit_gb)],
                       capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle worker failed (rc {r.returncode}): {r.stderr[-2000:]}")
    z = np.load(op)
    out = {}
    for task in tasks:
        n, ng, wb = (int(x) for x in z[f"{task}.meta"])
        ns = SimpleNamespace(n=n, n_groups=ng, wbits=wb)
        for f in FIELDS:
            setattr(ns, f, z[f"{task}.{f}"] if f"{task}.{f}" in z else None)
        out[task] = ns
    return out


if __name__ == "__main__":
    main()
