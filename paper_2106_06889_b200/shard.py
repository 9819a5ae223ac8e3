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
    got = gather_compacts(part, runner.rank, runner.world, getattr(runner, "collective_device", "cpu"))
    if runner.rank != 0:
        return None
    return combine(got, task, runner.num_words)


_FIELDS = ("group_off", "group_id", "group_key", "group_gram", "id", "key", "gram", "count")


def gather_compacts(part: Compact, rank: int, world: int, device="cpu"):
    """Rank 0 receives every rank's result arrays as flat int64 tensors
    (torch.distributed.gather: NCCL on GPUs, gloo on CPUs) — no pickling,
    one message per field sized by an all-gathered length table.  Returns the
    list of Compacts (rank order) on rank 0, None elsewhere."""
    import torch
    import torch.distributed as dist

    def arr(name):
        a = getattr(part, name)
        return np.zeros(0, np.int64) if a is None else np.asarray(a).astype(np.int64, copy=False).ravel()

    arrays = [arr(f) for f in _FIELDS]
    # per field: element count + 1 (0 = absent), then n, n_groups, wbits
    meta = [len(a) + 1 if getattr(part, f) is not None else 0 for f, a in zip(_FIELDS, arrays)]
    meta += [int(part.n), int(part.n_groups), int(part.wbits)]
    mt = torch.tensor(meta, dtype=torch.int64, device=device)
    metas = [torch.empty_like(mt) for _ in range(world)]
    dist.all_gather(metas, mt)
    metas = [m.cpu().numpy() for m in metas]
    out = [dict() for _ in range(world)] if rank == 0 else None
    for j, f in enumerate(_FIELDS):
        L = max(max(int(m[j]) - 1, 0) for m in metas)
        if L == 0 and all(m[j] == 0 for m in metas):
            continue
        buf = torch.zeros(max(L, 1), dtype=torch.int64, device=device)
        a = torch.from_numpy(arrays[j]).to(device)
        buf[:len(a)] = a
        bufs = [torch.empty_like(buf) for _ in range(world)] if rank == 0 else None
        dist.gather(buf, bufs, dst=0)
        if rank == 0:
            for r in range(world):
                nm = int(metas[r][j])
                out[r][f] = bufs[r][:nm - 1].cpu().numpy() if nm else None
    if rank != 0:
        return None
    res = []
    for r in range(world):
        m = metas[r]
        c = Compact(task=part.task, seq_len=part.seq_len, wbits=int(m[-1]), strategy=part.strategy,
                    n_groups=int(m[-2]), n=int(m[-3]))
        for f in _FIELDS:
            setattr(c, f, out[r].get(f))
        res.append(c)
    return res


class DeviceRunner:
    """`run_distributed` runner over a DeviceDag on this rank's device."""

    def __init__(self, dag, rank: int, world: int, ranges=None):
        self.dag, self.rank, self.world = dag, rank, world
        self.num_words = dag.info["num_words"]
        if ranges is None:
            ranges = shard_ranges(dag.dag_array("segment_token_counts"), world)
        self.file_lo, self.file_hi = ranges[rank]
        dag.set_files(self.file_lo, self.file_hi)
        self.collective_device = f"cuda:{dag.device}"

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


# ---------------------------------------------------------------------------
# one process, several devices (TraversalConfig.workers > 1)
# ---------------------------------------------------------------------------

class ShardedDag:
    """One corpus over `workers` file-range shards in ONE process
    (`TraversalConfig.workers`, engine.py:34-48 — the reference's worker
    count, here GPUs).  The DAG is built once (the given DeviceDag) and
    replicated to every shard's device with gt_clone (peer copies over
    NVLink; SURVEY §8e "uploads to GPU0 and broadcasts").  Shards run
    concurrently (one host thread each; ctypes releases the GIL).  Word
    count / sort: every shard's dense counts are summed on shard 0's device
    by one kernel reading the others through peer memory
    (gt_sum_word_counts), then assembled there (gt_assemble_counts); per-file
    tasks combine by file order (`combine`).  Devices default to
    ``i % device_count``: on a single GPU the shards share it (the logic and
    the results are those of the multi-GPU run)."""

    def __init__(self, dag, workers: int, devices=None):
        from .device import device_count
        if workers < 1:
            raise ValueError("workers must be >= 1")
        ndev = max(1, device_count())
        self.devices = list(devices) if devices else [i % ndev for i in range(workers)]
        if len(self.devices) != workers:
            raise ValueError("one device per worker")
        self.ranges = shard_ranges(dag.dag_array("segment_token_counts"), workers)
        self.grammar = dag.grammar
        self.num_words = dag.info["num_words"]
        self._info = dict(dag.info)
        self.shards = []
        try:
            for dev, (lo, hi) in zip(self.devices, self.ranges):
                s = dag.clone(dev)
                s.set_files(lo, hi)
                self.shards.append(s)
        except Exception:
            self.close()
            raise

    @property
    def info(self) -> dict:
        return self._info

    @property
    def num_files(self) -> int:
        return self._info["num_files"]

    @property
    def num_rules(self) -> int:
        return self._info["num_rules"]

    def _each(self, fn):
        from concurrent.futures import ThreadPoolExecutor
        if len(self.shards) == 1:
            return [fn(self.shards[0])]
        with ThreadPoolExecutor(len(self.shards)) as ex:
            return list(ex.map(fn, self.shards))

    def run(self, task_id: int, seq_len: int, strategy: int, file_set_width: int) -> Compact:
        from ._abi import TASK_IDS, TASK_NAMES
        task = TASK_NAMES[task_id]
        if task in WORD_TASKS_GLOBAL:
            self._each(lambda s: s.run(TASK_IDS["wordcount"], seq_len, strategy, file_set_width))
            s0 = self.shards[0]
            s0.sum_word_counts(self.shards)
            return s0.assemble_counts(s0.device_word_counts_ptr(), task_id)
        parts = self._each(lambda s: s.run(task_id, seq_len, strategy, file_set_width))
        return combine(parts, task, self.num_words)

    def run_many(self, task_ids, seq_len: int, strategy: int, file_set_width: int):
        return [self.run(t, seq_len, strategy, file_set_width) for t in task_ids]

    def close(self) -> None:
        for s in self.shards:
            s.close()
        self.shards = []

