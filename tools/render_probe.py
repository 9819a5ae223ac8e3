#!/usr/bin/env python3
"""Time native render/digest vs the Python render on large outputs (diagnostic)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200.corpus import compose, config_spec
    from paper_2106_06889_b200.native import NativeDict
    for spec in sys.argv[1:]:
        name, tasks = spec.split(":")
        blob, _ = compose(config_spec(name))
        dag = gt.DeviceDag(blob)
        nd = NativeDict(blob)
        for t in tasks.split(","):
            c = gt.run_compact(dag, t, gt.TraversalConfig(), 3)
            t0 = time.perf_counter()
            h, n = nd.digest(c)
            t1 = time.perf_counter()
            txt = nd.render(c)
            t2 = time.perf_counter()
            line = f"{name} {t:20s} records={c.n} bytes={n} digest {t1 - t0:.3f}s ({n / (t1 - t0) / 1e9:.2f} GB/s) render {t2 - t1:.3f}s"
            if c.n < 20_000_000:
                t3 = time.perf_counter()
                py = gt.render(gt._abi.to_container(c), dag.grammar.dictionary)
                t4 = time.perf_counter()
                assert py == txt
                line += f"  python render {t4 - t3:.2f}s (equal)"
            print(line, flush=True)
        dag.close()


if __name__ == "__main__":
    main()
