"""GPU vs CPU-oracle parity on composed corpora (bit-exact compact arrays),
plus size-independent properties at BASELINE config sizes.

The oracle (oracle/gt_oracle.c) is pinned to the reference by
tests/test_oracle_golden.py; here the device path must reproduce its
render-ordered arrays exactly.
"""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TASKS = ["wordcount", "sort", "invertedindex", "termvector", "seqcount", "rankedinvertedindex"]
FIELDS = ["group_off", "group_id", "group_key", "group_gram", "id", "key", "gram", "count"]


def same(a, b) -> bool:
    if a is None or b is None:
        return (a is None or len(a) == 0) and (b is None or len(b) == 0)
    return np.array_equal(np.asarray(a, dtype=np.int64), np.asarray(b, dtype=np.int64))


def assert_same(got, exp, what):
    assert got.n == exp.n and got.n_groups == exp.n_groups, (what, got.n, exp.n, got.n_groups, exp.n_groups)
    assert got.wbits == exp.wbits, what
    for f in FIELDS:
        assert same(getattr(got, f), getattr(exp, f)), (what, f)


def composed(name, scale, seed=None):
    from paper_2106_06889_b200.corpus import compose, config_spec
    return compose(config_spec(name, seed=seed, scale=scale))


CASES = [("c2", 0.002, None), ("c2", 0.01, 7), ("c3", 0.002, None), ("c3", 0.01, 11),
         ("c4", 0.0005, None), ("c5", 0.0002, None)]


@pytest.mark.parametrize("name,scale,seed", CASES)
def test_composed_all_tasks_match_oracle(name, scale, seed):
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    blob, stats = composed(name, scale, seed)
    dag = gt.DeviceDag(blob)
    ref = OracleDag(blob)
    assert dag.info["words"] == ref.info["words"] == stats["W"]
    for task in TASKS:
        lens = (2, 3, 4) if task in ("seqcount", "rankedinvertedindex") else (3,)
        for l in lens:
            for strategy in ("auto", "topdown", "bottomup"):
                cfg = gt.TraversalConfig(strategy=strategy)
                got = gt.run_compact(dag, task, cfg, l)
                exp = gt.run_compact(ref, task, gt.TraversalConfig(strategy="topdown"), l)
                assert_same(got, exp, (name, scale, task, l, strategy))
                if strategy == "bottomup" and task in ("wordcount", "sort", "invertedindex", "termvector"):
                    assert got.strategy == "bottomup"  # the pooled hash-table path ran
    dag.close()


def test_c2_full_wordcount_and_invertedindex_match_oracle():
    """BASELINE configs[1] at full size: the bench workload itself."""
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    blob, stats = composed("c2", 1.0)
    dag = gt.DeviceDag(blob)
    ref = OracleDag(blob)
    for task in ("wordcount", "invertedindex", "sort", "termvector"):
        got = gt.run_compact(dag, task, gt.TraversalConfig(), 3)
        exp = gt.run_compact(ref, task, gt.TraversalConfig(), 3)
        assert_same(got, exp, task)
    wc = gt.run_compact(dag, "wordcount", gt.TraversalConfig())
    assert int(wc.count.sum()) == stats["W"]  # weight conservation (test_acceptance criterion 3)
    dag.close()


def test_c2_full_sequence_properties():
    """Size-independent properties at full C2 size: per-file window totals equal
    tokens_f - (l-1); every gram's file list is sorted by (-count, file)."""
    import paper_2106_06889_b200 as gt
    blob, _ = composed("c2", 1.0)
    dag = gt.DeviceDag(blob)
    toks = dag.dag_array("segment_token_counts")
    sc = gt.run_compact(dag, "seqcount", gt.TraversalConfig(), 3)
    off = sc.group_off
    per_file = np.add.reduceat(sc.count, off[:-1]) if sc.n else np.zeros(len(toks))
    per_file = np.where(np.diff(off) > 0, per_file, 0)
    assert np.array_equal(per_file, np.maximum(toks - 2, 0))
    for f in range(len(toks)):
        c = sc.count[off[f]:off[f + 1]]
        assert np.all(c[:-1] >= c[1:])
    rii = gt.run_compact(dag, "rankedinvertedindex", gt.TraversalConfig(), 3)
    assert int(rii.count.sum()) == int(sc.count.sum())
    assert rii.n == sc.n
    dag.close()
