"""Multi-GPU execution by file-range shards.

Files are contiguous, splitter-delimited ranges of the root body
(`dag.py:107-128`) and every per-file output depends only on that file's
segment plus the shared DAG, so one process per GPU owns a contiguous file
range, balanced by uncompressed tokens (`segment_token_counts`,
`dag.py:88-104`).  The DAG is replicated (it is small next to 180 GB of HBM);
`gt_set_files` restricts seeds, root scans and per-file outputs to the owned
range.  Combination:

* word count / sort: the shards' dense u64[V] count vectors are summed with
  one all-reduce (NCCL over NVLink on GPUs; exact — integer sums) and rank 0
  assembles the render-ordered result on its device (`gt_assemble_counts`);
* term vector / sequence count: per-file groups are already in global file
  order, so rank 0 concatenates the shards' groups;
* inverted index / ranked inverted index: rank 0 merges the shards' groups
  by word / gram (file lists stay ascending; per-gram (file, count) lists are
  re-ordered by (-count, file) as `tasks.py:162-168` requires).

The combine functions are plain numpy over `Compact` results and are shared
by the GPU path and the CPU (gloo) tests.
"""

from __future__ import annotations

import numpy as np

from ._abi import Compact

WORD_TASKS_GLOBAL = ("wordcount", "sort")


def shard_ranges(tokens, n: int) -> list[tuple[int, int]]:
    """Token-balanced contiguous file ranges [(lo, hi)] for n shards (ranges
    may be empty when there are fewer files than shards)."""
    tokens = np.asarray(tokens, dtype=np.int64)
    F = len(tokens)
    if n < 1:
        raise ValueError("need at least one shard")
    cum = np.concatenate([[0], np.cumsum(tokens)])
    cuts = [0]
    for k in range(1, n):
        cuts.append(int(np.searchsorted(cum, cum[-1] * k / n, side="left")))
    cuts.append(F)
    cuts = np.maximum.accumulate(np.minimum(np.asarray(cuts), F))
    return [(int(cuts[i]), int(cuts[i + 1])) for i in range(n)]


# ---------------------------------------------------------------------------
# combination of per-shard compact results (rank order == file order)
# ---------------------------------------------------------------------------

def counts_dense(part: Compact, num_words: int) -> np.ndarray:
    """Dense u64[V] counts of a wordcount/sort result."""
    v = np.zeros(num_words, dtype=np.int64)
    if part.n:
        np.add.at(v, part.id, part.count)
    return v


def assemble_counts_host(dense: np.ndarray, task: str, seq_len: int = 3) -> Compact:
    """Host assembly of a word count / sort result from dense counts (used by
    the CPU tests; the GPU path assembles on the device)."""
    ids = np.flatnonzero(dense).astype(np.int64)
    cnt = dense[ids].astype(np.int64)
    if task == "sort" and len(ids):
        o = np.lexsort((ids, -cnt))
        ids, cnt = ids[o], cnt[o]
    return Compact(task=task, seq_len=seq_len, wbits=0, strategy="topdown", n_groups=0,
                   n=len(ids), id=ids, count=cnt)


def _cat(arrs):
    arrs = [a for a in arrs if a is not None]
    return np.concatenate(arrs) if arrs else None


def _grams_of(c: Compact, per_group: bool) -> np.ndarray:
    """(n, l) gram matrix (packed keys decoded) of records or groups."""
    return c.grams(per_group=per_group)


def _pack_like(template: Compact, grams: np.ndarray, per_group: bool, out: Compact) -> None:
    """Store grams in the template's representation (packed key or words)."""
    l = template.seq_len
    if template.wbits:
        k = np.zeros(len(grams), dtype=np.uint64)
        for j in range(l):
            k = (k << np.uint64(template.wbits)) | grams[:, j].astype(np.uint64)
        if per_group:
            out.group_key = k
        else:
            out.key = k
    else:
        flat = grams.reshape(-1).astype(np.int64)
        if per_group:
            out.group_gram = flat
        else:
            out.gram = flat


def combine(parts: list[Compact], task: str, num_words: int) -> Compact:
    """Combine per-shard results (in shard = file order) into the result of
    the whole corpus."""
    p0 = parts[0]
    l = p0.seq_len
    if task in WORD_TASKS_GLOBAL:
        dense = sum(counts_dense(p, num_words) for p in parts)
        return assemble_counts_host(dense, task, l)
    out = Compact(task=task, seq_len=l, wbits=p0.wbits, strategy=p0.strategy, n_groups=0, n=0)
    if task in ("termvector", "seqcount"):
        # groups are files: concatenate, shifting offsets
        offs, base = [], 0
        for p in parts:
            o = p.group_off if p.group_off is not None else np.zeros(1, np.int64)
            offs.append(o[:-1] + base)
            base += int(p.n)
        out.group_off = np.concatenate(offs + [np.asarray([base], np.int64)])
        out.n_groups = sum(int(p.n_groups) for p in parts)
        out.n = base
        out.id = _cat([p.id for p in parts])
        out.key = _cat([p.key for p in parts])
        out.gram = _cat([p.gram for p in parts])
        out.count = _cat([p.count for p in parts])
        return out
    if task == "invertedindex":
        # (word, file) records; shards hold ascending disjoint file ranges
        words = _cat([np.repeat(p.group_id, np.diff(p.group_off)) for p in parts if p.n])
        files = _cat([p.id for p in parts if p.n])
        if words is None:
            out.group_off = np.zeros(1, np.int64)
            out.group_id = np.zeros(0, np.int64)
            out.id = np.zeros(0, np.int64)
            return out
        o = np.argsort(words, kind="stable")
        words, files = words[o], files[o]
        gid, start = np.unique(words, return_index=True)
        out.group_id = gid
        out.group_off = np.concatenate([start, [len(words)]]).astype(np.int64)
        out.n_groups, out.n, out.id = len(gid), len(words), files
        return out
    if task == "rankedinvertedindex":
        grams = [np.repeat(_grams_of(p, True), np.diff(p.group_off), axis=0) for p in parts if p.n]
        if not grams:
            out.group_off = np.zeros(1, np.int64)
            out.id = np.zeros(0, np.int64)
            out.count = np.zeros(0, np.int64)
            _pack_like(p0, np.zeros((0, l), np.int64), True, out)
            return out
        g = np.concatenate(grams)
        files = _cat([p.id for p in parts if p.n])
        cnt = _cat([p.count for p in parts if p.n])
        # order: gram ascending, then (-count, file)
        keys = [files, -cnt] + [g[:, j] for j in range(l - 1, -1, -1)]
        o = np.lexsort(keys)
        g, files, cnt = g[o], files[o], cnt[o]
        head = np.ones(len(g), dtype=bool)
        head[1:] = np.any(g[1:] != g[:-1], axis=1)
        start = np.flatnonzero(head)
        out.group_off = np.concatenate([start, [len(g)]]).astype(np.int64)
        out.n_groups, out.n = len(start), len(g)
        out.id, out.count = files, cnt
        _pack_like(p0, g[start], True, out)
        return out
    raise ValueError(f"unknown task {task!r}")


# ---------------------------------------------------------------------------
# distributed driver (one process per device, torch.distributed plumbing)
# ---------------------------------------------------------------------------

def run_distributed(runner, task: str, seq_len: int = 3, strategy: int = 0,
                    file_set_width: int = 64):
    """Run `task` on this rank's shard and combine on rank 0.

    `runner` provides: `rank`, `world`, `num_words`, `run(task_id, seq_len,
    strategy, fsw) -> Compact` for its own file range, `counts_tensor()` (the
    shard's dense int64[V] counts as a torch tensor on the collective's
    device, valid after a wordcount/sort run) and `assemble(tensor, task) ->
    Compact`.  Returns the combined Compact on rank 0, None elsewhere."""
    import torch.distributed as dist

    from ._abi import TASK_IDS

    part = runner.run(TASK_IDS["wordcount" if task in WORD_TASKS_GLOBAL else task], seq_len,
                      strategy, file_set_width)
    if task in WORD_TASKS_GLOBAL:
        t = runner.counts_tensor()
        dist.all_reduce(t)  # exact: integer sums
        return runner.assemble(t, task) if runner.rank == 0 else None
    got = [None] * runner.world if runner.rank == 0 else None
    dist.gather_object(part, got, dst=0)
    if runner.rank != 0:
        return None
    return combine(got, task, runner.num_words)


class DeviceRunner:
    """`run_distributed` runner over a DeviceDag on this rank's device."""

    def __init__(self, dag, rank: int, world: int, ranges=None):
        self.dag, self.rank, self.world = dag, rank, world
        self.num_words = dag.info["num_words"]
        if ranges is None:
            ranges = shard_ranges(dag.dag_array("segment_token_counts"), world)
        self.file_lo, self.file_hi = ranges[rank]
        dag.set_files(self.file_lo, self.file_hi)

    def run(self, task_id, seq_len, strategy, fsw):
        return self.dag.run(task_id, seq_len, strategy, fsw)

    def counts_tensor(self):
        import torch
        ptr = self.dag.device_word_counts_ptr()
        V = self.num_words

        class _CAI:  # __cuda_array_interface__ view of the library's u64[V]
            __cuda_array_interface__ = {"shape": (V,), "typestr": "<i8", "data": (ptr, False),
                                        "version": 3}
        return torch.as_tensor(_CAI(), device=f"cuda:{self.dag.device}").clone()

    def assemble(self, t, task):
        from ._abi import TASK_IDS
        return self.dag.assemble_counts(t.data_ptr(), TASK_IDS[task])
