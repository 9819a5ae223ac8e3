"""The single-parent contraction of the top-down pass (contract.cu): for
every rule its head H (the nearest ancestor with more than one non-root
parent edge or a root reference), multiplier M (w(r) = M(r)·w(H(r))) and
contracted level L' (heads: 1 + max over parents of L'(H(parent)), the root
0; singles: their head's), against a numpy restatement over the device's own
(reference-pinned) parent CSR and top-down levels; and the word tasks run
over the heads-only lists (built on a DAG's second top-down run) == the
first, full run == the oracle."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import fixture_names, gtdc
from test_gpu_parity import composed

pytestmark = pytest.mark.gpu


def expected_contraction(dag):
    po = dag.dag_array("par_off")
    pid = dag.dag_array("par_ids")
    pf = dag.dag_array("par_freqs")
    td = dag.dag_array("td_level")
    R = len(td)
    npar = np.diff(po)
    child = np.repeat(np.arange(R), npar)
    nonroot = np.bincount(child[pid != 0], minlength=R)
    rootref = np.zeros(R, bool)
    rootref[child[pid == 0]] = True
    single = (nonroot == 1) & ~rootref
    single[0] = False
    H = np.arange(R)
    M = np.ones(R, np.int64)
    L = np.zeros(R, np.int64)
    for c in np.argsort(td, kind="stable"):
        if c == 0:
            continue
        ps = pid[po[c]:po[c + 1]]
        fs = pf[po[c]:po[c + 1]]
        keep = ps != 0
        ps, fs = ps[keep], fs[keep]
        if single[c]:
            p = ps[0]
            H[c], M[c], L[c] = H[p], M[p] * fs[0], L[p]
        else:
            L[c] = 1 + max((L[p] for p in ps), default=0)
    return H, M, L


def _check(dag):
    head_t = dag.dag_array("cont_head")  # tid space (builds the contraction)
    H, M, L = expected_contraction(dag)
    fits = M < (1 << 32)
    if head_t.size == 0:  # nothing to contract, or a multiplier (or f·M) outgrew 32 bits
        assert len(H) < 2 or not fits.all() or _edge_overflow(dag, H, M)
        assert not dag.refresh_info()["load_flags"] & 4
        return
    assert dag.refresh_info()["load_flags"] & 4
    tid = dag.dag_array("tid")
    rule_of = np.argsort(tid)
    assert np.array_equal(rule_of[head_t[tid]], H)
    assert np.array_equal(dag.dag_array("cont_mult")[tid], M)
    assert np.array_equal(dag.dag_array("cont_level")[tid], L)
    # tid': heads by (L', tid), singles after every head
    row = dag.dag_array("cont_row")[tid]
    heads = np.flatnonzero(H == np.arange(len(H)))
    order = heads[np.lexsort((tid[heads], L[heads]))]
    assert np.array_equal(row[order], np.arange(len(heads)))
    assert (row[H != np.arange(len(H))] >= len(heads)).all()


def _edge_overflow(dag, H, M):
    """some f·M(parent) of an edge or f·M(rule) of an own pair needs 64 bits"""
    pid, pf = dag.dag_array("par_ids"), dag.dag_array("par_freqs")
    if (pf.astype(object) * M[pid].astype(object) >= (1 << 32)).any():
        return True
    oo, of = dag.dag_array("own_off"), dag.dag_array("own_freqs")
    rule = np.repeat(np.arange(len(oo) - 1), np.diff(oo))
    return bool((of.astype(object) * M[rule].astype(object) >= (1 << 32)).any())


@pytest.mark.parametrize("name", fixture_names())
def test_contraction_on_fixtures(name):
    import paper_2106_06889_b200 as gt
    try:
        dag = gt.DeviceDag(gtdc(name))
    except gt.GtadocError:
        pytest.skip("invalid grammar")
    with dag:
        _check(dag)


@pytest.mark.parametrize("src", ["c2@0.05", "c3@0.02", "c4@0.001", "c5@0.001"])
def test_contraction_on_composed(src):
    import paper_2106_06889_b200 as gt
    name, sc = src.split("@")
    with gt.DeviceDag(composed(name, float(sc))[0]) as dag:
        _check(dag)


WORD_TASKS = ["wordcount", "sort", "invertedindex", "termvector"]


@pytest.mark.parametrize("src", ["c2@0.01", "c3@0.01", "c4@0.0005", "c5@0.0003"])
def test_second_run_is_contracted_and_identical(src):
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    from test_gpu_parity import assert_same
    name, sc = src.split("@")
    blob = composed(name, float(sc))[0]
    ref = OracleDag(blob)
    cfg = gt.TraversalConfig(strategy="topdown")
    with gt.DeviceDag(blob) as dag:
        first = gt.run_compact(dag, "wordcount", cfg, 3)
        assert not dag.refresh_info()["load_flags"] & 4  # a one-shot query keeps the full lists
        assert_same(first, gt.run_compact(ref, "wordcount", cfg, 3), (src, "wordcount", "full"))
        second = gt.run_compact_many(dag, WORD_TASKS, cfg, 3)
        assert dag.refresh_info()["load_flags"] & 4
        third = [gt.run_compact(dag, t, cfg, 3) for t in WORD_TASKS]
        for t, b, c in zip(WORD_TASKS, second, third):
            exp = gt.run_compact(ref, t, cfg, 3)
            assert_same(b, exp, (src, t, "contracted"))
            assert_same(c, exp, (src, t, "contracted, single task"))


@pytest.mark.parametrize("src", ["c4@0.2", "c5@0.12"])
def test_large_grammar_shared_pair_pass(src):
    """> 4·10^6 own pairs: once contracted, word count + inverted index share
    one pair pass (level launch, full-occupancy word reduce, compaction
    launch) instead of two separate passes; both equal the oracle."""
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    from test_gpu_parity import assert_same
    name, sc = src.split("@")
    blob = composed(name, float(sc))[0]
    cfg = gt.TraversalConfig(strategy="topdown")
    tasks = ["wordcount", "invertedindex"]
    with gt.DeviceDag(blob) as dag:
        assert dag.info["own_pairs"] > 4 << 20
        first = gt.run_compact_many(dag, tasks, cfg, 3)  # separate passes over every rule
        second = gt.run_compact_many(dag, tasks, cfg, 3)  # builds the contraction, shared pass
        assert dag.refresh_info()["load_flags"] & 4
        third = gt.run_compact_many(dag, tasks, cfg, 3)
    ref = OracleDag(blob)
    for t, a, b, c in zip(tasks, first, second, third):
        exp = gt.run_compact(ref, t, cfg, 3)
        assert_same(a, exp, (src, t, "full"))
        assert_same(b, exp, (src, t, "contracted"))
        assert_same(c, exp, (src, t, "contracted again"))


def test_large_contracted_pass_on_file_shards():
    """The shared large-grammar pass after gt_set_files: the contracted seeds
    follow the owned file range, and the shards' word counts (summed) and
    inverted indexes (combined in file order) equal the whole corpus."""
    import torch

    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200._abi import TASK_IDS
    from paper_2106_06889_b200.shard import DeviceRunner, combine
    from test_shard_cpu import same_compact
    blob = composed("c4", 0.2)[0]
    cfg = gt.TraversalConfig(strategy="topdown")
    with gt.DeviceDag(blob) as dag:
        V = dag.info["num_words"]
        gt.run_compact_many(dag, ["wordcount", "invertedindex"], cfg, 3)
        whole = gt.run_compact_many(dag, ["wordcount", "invertedindex"], cfg, 3)  # contracted
        assert dag.refresh_info()["load_flags"] & 4
        acc = torch.zeros(V, dtype=torch.int64, device="cuda")
        parts = []
        for rank in range(3):
            r = DeviceRunner(dag, rank, 3)
            wc, ii = dag.run_many([TASK_IDS["wordcount"], TASK_IDS["invertedindex"]], 3, 0, 64)
            acc += r.counts_tensor()
            parts.append(ii)
        same_compact(r.assemble(acc, "wordcount"), whole[0])
        same_compact(combine(parts, "invertedindex", V), whole[1])
        dag.set_files(0, 1 << 62)
        same_compact(gt.run_compact_many(dag, ["wordcount", "invertedindex"], cfg, 3)[1], whole[1])


@pytest.mark.parametrize("policy,expect", [("0", [False, False, False]), ("2", [True, True, True]),
                                           ("1", [False, True, True])])
def test_contraction_build_policy(policy, expect):
    """GT_CONTRACT=0 never builds the contraction, 2 on the first run, the
    default (1) on the DAG's second public run call (read once per process:
    a subprocess per policy)."""
    import json
    import os
    import subprocess
    import sys
    code = (
        "import json, sys\n"
        "sys.path.insert(0, '.')\n"
        "import paper_2106_06889_b200 as gt\n"
        "from paper_2106_06889_b200.corpus import compose, config_spec\n"
        "blob, _ = compose(config_spec('c2', scale=0.01))\n"
        "dag = gt.DeviceDag(blob)\n"
        "ref = gt.run_compact(dag, 'wordcount', gt.TraversalConfig())\n"
        "flags = [bool(dag.refresh_info()['load_flags'] & 4)]\n"
        "for _ in range(2):\n"
        "    c = gt.run_compact(dag, 'wordcount', gt.TraversalConfig())\n"
        "    assert (c.id == ref.id).all() and (c.count == ref.count).all()\n"
        "    flags.append(bool(dag.refresh_info()['load_flags'] & 4))\n"
        "print(json.dumps(flags))\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, GT_CONTRACT=policy),
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1]) == expect
