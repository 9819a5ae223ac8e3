"""ctypes mirror of include/gtadoc_b200.h and the view -> container conversion.

Shared by the product facade (tasks.py, over libgtadoc_b200.so) and by the
test-only CPU oracle wrapper (oracle/oracle.py), which exports the same
`gt_view` layout under a `gto_` prefix.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from .errors import CorruptionError, FormatError, ResourceError, UsageError

GT_OK, GT_E_USAGE, GT_E_RESOURCE, GT_E_FORMAT, GT_E_CORRUPTION, GT_E_DEVICE = range(6)
TASK_IDS = {
    "wordcount": 0,
    "sort": 1,
    "invertedindex": 2,
    "termvector": 3,
    "seqcount": 4,
    "rankedinvertedindex": 5,
}
TASK_NAMES = tuple(TASK_IDS)
STRATEGY_IDS = {"auto": 0, "topdown": 1, "bottomup": 2}
STRATEGY_NAMES = {v: k for k, v in STRATEGY_IDS.items()}
STRATEGY_NAMES[3] = "topdown-sparse"  # GT_TOPDOWN_SPARSE (reported, not requested)

_EXC = {
    GT_E_USAGE: UsageError,
    GT_E_RESOURCE: ResourceError,
    GT_E_FORMAT: FormatError,
    GT_E_CORRUPTION: CorruptionError,
    GT_E_DEVICE: ResourceError,
}


def raise_for_status(status: int, message: str) -> None:
    if status != GT_OK:
        raise _EXC.get(status, ResourceError)(message)


class GtInfo(C.Structure):
    _fields_ = [
        ("num_words", C.c_uint64),
        ("num_splitters", C.c_uint64),
        ("num_rules", C.c_uint64),
        ("num_files", C.c_uint64),
        ("total_elements", C.c_uint64),
        ("root_len", C.c_uint64),
        ("sub_pairs", C.c_uint64),
        ("own_pairs", C.c_uint64),
        ("words", C.c_uint64),
        ("depth", C.c_int64),
        ("td_levels", C.c_int64),
        ("bu_levels", C.c_int64),
        ("device_bytes", C.c_uint64),
        ("init_ms", C.c_double),
        ("td_edges", C.c_uint64),
        ("load_flags", C.c_uint64),
    ]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


_P64 = C.POINTER(C.c_uint64)
_P32 = C.POINTER(C.c_uint32)


class GtView(C.Structure):
    _fields_ = [
        ("task", C.c_int32),
        ("seq_len", C.c_int32),
        ("wbits", C.c_int32),
        ("strategy", C.c_int32),
        ("n_groups", C.c_uint64),
        ("group_off", _P64),
        ("group_id", _P32),
        ("group_key", _P64),
        ("group_gram", _P32),
        ("n", C.c_uint64),
        ("id", _P32),
        ("key", _P64),
        ("gram", _P32),
        ("count", _P64),
        ("device_ms", C.c_double),
        ("d2h_ms", C.c_double),
        ("total_ms", C.c_double),
        ("d2h_bytes", C.c_uint64),
        ("kernel_launches", C.c_uint64),
        ("count32", _P32),      # ABI 2: narrowed copies (count / group_off NULL then)
        ("group_off32", _P32),
        ("id_narrow", C.c_void_p),  # ABI 3: ids id_bytes (1 / 2) wide (id NULL then)
        ("id_bytes", C.c_int32),
        ("reserved_", C.c_int32),
    ]


def _arr(ptr, n: int, dtype):
    if not ptr or n == 0:
        return None if not ptr else np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


@dataclass
class Compact:
    """Compact, render-ordered result arrays (one gt_view, copied)."""

    task: str
    seq_len: int
    wbits: int
    strategy: str
    n_groups: int
    n: int
    group_off: np.ndarray | None = None
    group_id: np.ndarray | None = None
    group_key: np.ndarray | None = None
    group_gram: np.ndarray | None = None
    id: np.ndarray | None = None
    key: np.ndarray | None = None
    gram: np.ndarray | None = None
    count: np.ndarray | None = None
    timings: dict = field(default_factory=dict)

    def grams(self, per_group: bool = False) -> np.ndarray:
        """(n, seq_len) word-id matrix of the record (or group) grams; decodes
        packed keys big-endian by position (sequence.py:244-256)."""
        key = self.group_key if per_group else self.key
        gram = self.group_gram if per_group else self.gram
        n = self.n_groups if per_group else self.n
        l = self.seq_len
        if self.wbits == 0:
            return (gram if gram is not None else np.zeros(0, np.uint32)).reshape(n, l).astype(np.int64)
        mask = (1 << self.wbits) - 1
        shifts = np.asarray([(l - 1 - j) * self.wbits for j in range(l)], dtype=np.uint64)
        k = key.astype(np.uint64).reshape(-1, 1) if n else np.zeros((0, 1), np.uint64)
        return ((k >> shifts) & np.uint64(mask)).astype(np.int64)


def compact_from_view(v: GtView) -> Compact:
    task = TASK_NAMES[v.task]
    ng, n, l = int(v.n_groups), int(v.n), int(v.seq_len)
    c = Compact(task=task, seq_len=l, wbits=int(v.wbits), strategy=STRATEGY_NAMES.get(int(v.strategy), "?"),
                n_groups=ng, n=n)
    c.group_off = (_arr(v.group_off, ng + 1, np.int64) if v.group_off else
                   _arr(v.group_off32, ng + 1, np.int64) if v.group_off32 else None)
    c.group_id = _arr(v.group_id, ng, np.int64)
    c.group_key = _arr(v.group_key, ng, np.uint64)
    c.group_gram = _arr(v.group_gram, ng * l, np.int64)
    if v.id_narrow:
        cty = C.c_uint8 if v.id_bytes == 1 else C.c_uint16
        c.id = _arr(C.cast(v.id_narrow, C.POINTER(cty)), n, np.int64)
    else:
        c.id = _arr(v.id, n, np.int64)
    c.key = _arr(v.key, n, np.uint64)
    c.gram = _arr(v.gram, n * l, np.int64)
    c.count = _arr(v.count, n, np.int64) if v.count else _arr(v.count32, n, np.int64)
    c.timings = dict(device_ms=v.device_ms, d2h_ms=v.d2h_ms, total_ms=v.total_ms,
                     d2h_bytes=int(v.d2h_bytes), kernel_launches=int(v.kernel_launches))
    return c


def to_container(c: Compact):
    """Build the reference's output container (tasks.py:61-88) from arrays."""
    from .tasks import (InvertedIndex, RankedInvertedIndex, SequenceCounts, SortedWords,
                        TermVectors, WordCounts)
    ids = c.id.tolist() if c.id is not None else []
    cnt = c.count.tolist() if c.count is not None else []
    off = c.group_off.tolist() if c.group_off is not None else [0]
    if c.task == "wordcount":
        return WordCounts(dict(zip(ids, cnt)))
    if c.task == "sort":
        return SortedWords(list(zip(ids, cnt)))
    if c.task == "invertedindex":
        gid = c.group_id.tolist() if c.group_id is not None else []
        return InvertedIndex({gid[g]: ids[off[g]:off[g + 1]] for g in range(c.n_groups)})
    if c.task == "termvector":
        pairs = list(zip(ids, cnt))
        return TermVectors([pairs[off[f]:off[f + 1]] for f in range(c.n_groups)])
    if c.task == "seqcount":
        grams = [tuple(g) for g in c.grams().tolist()]
        return SequenceCounts([dict(zip(grams[off[f]:off[f + 1]], cnt[off[f]:off[f + 1]]))
                               for f in range(c.n_groups)])
    grams = [tuple(g) for g in c.grams(per_group=True).tolist()]
    pairs = list(zip(ids, cnt))
    return RankedInvertedIndex({grams[g]: pairs[off[g]:off[g + 1]] for g in range(c.n_groups)})
