"""Multi-GPU host logic on CPU: shard ranges, combination of per-shard results,
and the torch.distributed driver at world size 2 over gloo.

Per-shard results are derived from the oracle's whole-corpus results (the
oracle has no file ranges): a shard's word counts are the sum of its files'
term vectors, its per-file groups are the full result's groups of its files.
The GPU test (tests/test_gpu_shards.py) checks the device shards themselves.
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import gtdc

TASKS = ["wordcount", "sort", "invertedindex", "termvector", "seqcount", "rankedinvertedindex"]
FIELDS = ["group_off", "group_id", "group_key", "group_gram", "id", "key", "gram", "count"]


def same_compact(a, b):
    assert a.n == b.n and a.n_groups == b.n_groups, (a.n, b.n, a.n_groups, b.n_groups)
    for f in FIELDS:
        x, y = getattr(a, f), getattr(b, f)
        if x is None or y is None:
            assert (x is None or len(x) == 0) and (y is None or len(y) == 0), f
        else:
            assert np.array_equal(np.asarray(x, np.int64), np.asarray(y, np.int64)), f


def oracle_results(blob, l=3):
    import paper_2106_06889_b200 as gt
    from oracle.oracle import OracleDag
    ref = OracleDag(blob, workers=2)
    out = {t: gt.run_compact(ref, t, gt.TraversalConfig(), l) for t in TASKS}
    toks = ref.dag_array("segment_token_counts")
    V = ref.info["num_words"]
    ref.close()
    return out, toks, V


def split(full: dict, task: str, lo: int, hi: int, V: int):
    """The result a shard owning files [lo, hi) produces."""
    from paper_2106_06889_b200._abi import Compact
    from paper_2106_06889_b200.shard import assemble_counts_host
    c = full[task]
    if task in ("wordcount", "sort"):
        tv = full["termvector"]
        a, b = tv.group_off[lo], tv.group_off[hi]
        dense = np.zeros(V, np.int64)
        np.add.at(dense, tv.id[a:b], tv.count[a:b])
        return assemble_counts_host(dense, "wordcount", c.seq_len)
    p = Compact(task=task, seq_len=c.seq_len, wbits=c.wbits, strategy=c.strategy, n_groups=0, n=0)
    if task in ("termvector", "seqcount"):
        a, b = c.group_off[lo], c.group_off[hi]
        p.group_off = c.group_off[lo:hi + 1] - a
        p.n_groups, p.n = hi - lo, int(b - a)
        p.id = c.id[a:b] if c.id is not None else None
        p.count = c.count[a:b]
        p.key = c.key[a:b] if c.key is not None else None
        p.gram = c.gram[a * c.seq_len:b * c.seq_len] if c.gram is not None else None
        return p
    # grouped by word / gram: keep records whose file is in range
    keep = (c.id >= lo) & (c.id < hi)
    gidx = np.repeat(np.arange(c.n_groups), np.diff(c.group_off))[keep]
    p.id = c.id[keep]
    if c.count is not None:
        p.count = c.count[keep]
    groups, start = np.unique(gidx, return_index=True)
    p.group_off = np.concatenate([start, [len(gidx)]]).astype(np.int64)
    p.n_groups, p.n = len(groups), int(keep.sum())
    if c.group_id is not None:
        p.group_id = c.group_id[groups]
    if c.group_key is not None:
        p.group_key = c.group_key[groups]
    if c.group_gram is not None:
        l = c.seq_len
        p.group_gram = c.group_gram.reshape(-1, l)[groups].reshape(-1) if len(groups) else c.group_gram[:0]
    return p


def test_shard_ranges_cover_and_balance():
    from paper_2106_06889_b200.shard import shard_ranges
    rng = np.random.default_rng(0)
    for F in (1, 2, 7, 100, 1000):
        toks = rng.integers(0, 1000, size=F)
        for n in (1, 2, 3, 8):
            r = shard_ranges(toks, n)
            assert len(r) == n and r[0][0] == 0 and r[-1][1] == F
            assert all(a[1] == b[0] for a, b in zip(r, r[1:]))
            assert all(lo <= hi for lo, hi in r)
            loads = [int(toks[lo:hi].sum()) for lo, hi in r]
            assert max(loads) <= toks.sum() / n + toks.max() + 1


@pytest.mark.parametrize("name", ["g1", "many_files_70", "fuzz_03", "composed_2"])
@pytest.mark.parametrize("nshards", [2, 3])
def test_combine_of_shard_results_equals_whole_corpus(name, nshards):
    from paper_2106_06889_b200.shard import combine, shard_ranges
    full, toks, V = oracle_results(gtdc(name))
    ranges = shard_ranges(toks, nshards)
    for task in TASKS:
        parts = [split(full, task, lo, hi, V) for lo, hi in ranges]
        same_compact(combine(parts, task, V), full[task])


class _CpuRunner:
    """run_distributed runner whose shard results come from `split`."""

    def __init__(self, full, rank, world, ranges, V):
        self.full, self.rank, self.world, self.num_words = full, rank, world, V
        self.lo, self.hi = ranges[rank]
        self._last = None

    def run(self, task_id, seq_len, strategy, fsw):
        from paper_2106_06889_b200._abi import TASK_NAMES
        self._last = split(self.full, TASK_NAMES[task_id], self.lo, self.hi, self.num_words)
        return self._last

    def counts_tensor(self):
        import torch
        from paper_2106_06889_b200.shard import counts_dense
        return torch.from_numpy(counts_dense(self._last, self.num_words))

    def assemble(self, t, task):
        from paper_2106_06889_b200.shard import assemble_counts_host
        return assemble_counts_host(t.numpy(), task)


def _worker(rank, world, port, name, q):
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    import torch.distributed as dist
    from paper_2106_06889_b200.shard import run_distributed, shard_ranges
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full, toks, V = oracle_results(gtdc(name))
        runner = _CpuRunner(full, rank, world, shard_ranges(toks, world), V)
        for task in TASKS:
            got = run_distributed(runner, task)
            if rank == 0:
                same_compact(got, full[task])
            else:
                assert got is None
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("name", ["many_files_70", "composed_1"])
def test_gloo_world2_distributed_driver(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
