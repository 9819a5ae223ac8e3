"""Device file-range shards (gt_set_files) combined == the whole-corpus result,
for every task, on one GPU (the multi-GPU run differs only in where the
shards live).  Word counts are combined on the device like the NCCL
all-reduce: the shards' dense count vectors are summed in a torch tensor and
assembled with gt_assemble_counts."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import gtdc
from test_shard_cpu import TASKS, same_compact

pytestmark = pytest.mark.gpu


def composed(name, scale):
    from paper_2106_06889_b200.corpus import compose, config_spec
    return compose(config_spec(name, scale=scale))[0]


@pytest.mark.parametrize("src", ["g1", "many_files_70", "composed_2", "c2@0.003", "c3@0.003"])
@pytest.mark.parametrize("nshards", [2, 3, 5])
@pytest.mark.parametrize("strategy", ["auto", "bottomup"])
def test_device_shards_combine_to_whole(src, nshards, strategy):
    import torch

    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200._abi import TASK_IDS
    from paper_2106_06889_b200.shard import DeviceRunner, combine
    blob = composed(*src.split("@")[0:1], float(src.split("@")[1])) if "@" in src else gtdc(src)
    dag = gt.DeviceDag(blob)
    V = dag.info["num_words"]
    sid = gt._abi.STRATEGY_IDS[strategy]
    for l in (2, 3):
        full = {t: gt.run_compact(dag, t, gt.TraversalConfig(), l) for t in TASKS}
        for task in TASKS:
            if task in ("wordcount", "sort"):
                acc = torch.zeros(V, dtype=torch.int64, device="cuda")
                for rank in range(nshards):
                    r = DeviceRunner(dag, rank, nshards)
                    r.run(TASK_IDS["wordcount"], l, sid, 64)
                    acc += r.counts_tensor()
                got = r.assemble(acc, task)
            else:
                parts = []
                for rank in range(nshards):
                    r = DeviceRunner(dag, rank, nshards)
                    parts.append(r.run(TASK_IDS[task], l, sid, 64))
                got = combine(parts, task, V)
            same_compact(got, full[task])
        dag.set_files(0, 1 << 62)
    dag.close()


def test_empty_shard_outputs_are_empty():
    import paper_2106_06889_b200 as gt
    with gt.DeviceDag(gtdc("many_files_70")) as dag:
        dag.set_files(5, 5)
        for task in TASKS:
            c = gt.run_compact(dag, task, gt.TraversalConfig(), 3)
            assert c.n == 0, task
        dag.set_files(0, 1 << 62)
        assert gt.run_compact(dag, "wordcount", gt.TraversalConfig()).n > 0


# ---------------------------------------------------------------------------
# TraversalConfig.workers > 1 through the library: the DAG replicated with
# gt_clone, shards run concurrently, word counts summed through peer memory
# (gt_sum_word_counts), per-file results combined in file order
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("src", ["g1", "many_files_70", "composed_2", "c2@0.003", "c3@0.003"])
@pytest.mark.parametrize("workers", [2, 3, 4])
def test_workers_config_matches_single_device(src, workers):
    import paper_2106_06889_b200 as gt
    blob = composed(*src.split("@")[0:1], float(src.split("@")[1])) if "@" in src else gtdc(src)
    with gt.DeviceDag(blob) as dag:
        for l in (2, 3):
            one = gt.run_compact_many(dag, TASKS, gt.TraversalConfig(), l)
            many = gt.run_compact_many(dag, TASKS, gt.TraversalConfig(workers=workers), l)
            for task, a, b in zip(TASKS, many, one):
                same_compact(a, b)
            # the reference containers through run_task
            for task in ("wordcount", "invertedindex"):
                assert gt.run_task(dag, task, gt.TraversalConfig(workers=workers)) == \
                    gt.run_task(dag, task, gt.TraversalConfig())


def test_clone_replicates_every_dag_array():
    import paper_2106_06889_b200 as gt
    with gt.DeviceDag(gtdc("many_files_70")) as dag:
        c = dag.clone(0)
        try:
            for name in ("own_ids", "own_freqs", "own_off", "sub_ids", "sub_off", "par_ids", "par_off",
                         "exp_len", "td_level", "bu_level", "segments", "segment_token_counts"):
                assert np.array_equal(c.dag_array(name), dag.dag_array(name)), name
            assert c.info["words"] == dag.info["words"]
        finally:
            c.close()


def test_sum_word_counts_is_the_corpus_total():
    import paper_2106_06889_b200 as gt
    from paper_2106_06889_b200._abi import TASK_IDS
    from paper_2106_06889_b200.shard import shard_ranges
    with gt.DeviceDag(composed("c2", 0.003)) as dag:
        full = gt.run_compact(dag, "wordcount", gt.TraversalConfig())
        toks = dag.dag_array("segment_token_counts")
        shards = []
        try:
            for lo, hi in shard_ranges(toks, 3):
                s = dag.clone(0)
                s.set_files(lo, hi)
                s.run(TASK_IDS["wordcount"], 3, 0, 64)
                shards.append(s)
            shards[1].sum_word_counts(shards)  # dst may be any shard
            got = shards[1].assemble_counts(shards[1].device_word_counts_ptr(), TASK_IDS["wordcount"])
            same_compact(got, full)
        finally:
            for s in shards:
                s.close()
