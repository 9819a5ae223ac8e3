"""Concurrency stress of the device hash-table insert path (the pooled
bottom-up tables), the analogue of the reference's add_batch tests
(pkg/tests/test_table.py:145-164, test_acceptance.py:236-268): many warps
inserting Zipf-duplicated keys concurrently must equal a sequential replay,
every key at most once in the table, and overflow must raise ResourceError
(the reference's FULL status)."""

from __future__ import annotations

from collections import Counter

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,vocab,cap", [(1_000_000, 50_000, 1 << 17), (1_000_000, 64, 128),
                                         (200_000, 100_000, 1 << 18), (1, 1, 2), (0, 1, 2)])
def test_concurrent_inserts_equal_sequential_replay(n, vocab, cap):
    from paper_2106_06889_b200.device import table_add_batch
    rng = np.random.default_rng(n + vocab)
    keys = np.minimum(rng.zipf(1.2, size=n), vocab).astype(np.uint32) - 1 if n else np.zeros(0, np.uint32)
    deltas = rng.integers(1, 1000, size=n, dtype=np.uint64)
    got, slots, _ = table_add_batch(keys, deltas, cap)
    exp = Counter()
    for k, d in zip(keys.tolist(), deltas.tolist()):
        exp[k] += d
    assert got == dict(exp)
    occ = slots[slots != 0xFFFFFFFF]
    assert len(occ) == len(set(occ.tolist()))  # each key in one slot


def test_overflow_raises_resource_error():
    from paper_2106_06889_b200 import ResourceError
    from paper_2106_06889_b200.device import table_add_batch
    with pytest.raises(ResourceError):
        table_add_batch(np.arange(100, dtype=np.uint32), np.ones(100, np.uint64), 64)
