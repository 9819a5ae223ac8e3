"""Deterministic corpus generators shared by tools/make_golden.py (which ran
the REFERENCE Sequitur on them to produce tests/golden/grammars) and the
native-compressor tests (which must reproduce those bytes).  No reference
import: the generators follow the reference test suite's distributions
(pkg/tests/conftest.py:31-48, test_acceptance.py:54-72) with numpy only."""

from __future__ import annotations

import numpy as np


def corpus_tokens(rng, *, max_files=64, max_tokens=100_000, max_vocab=5000, min_files=1):
    """Same distribution as the reference's pkg/tests/conftest.py:31-48."""
    num_files = int(rng.integers(min_files, max_files + 1))
    vocab_size = int(rng.integers(1, max_vocab + 1))
    vocab = [f"w{i}" for i in range(vocab_size)]
    total = int(rng.integers(0, max_tokens + 1))
    files = []
    remaining = total
    for i in range(num_files):
        n = remaining if i == num_files - 1 else int(rng.integers(0, remaining + 1))
        n = min(n, max(0, remaining))
        ranks = np.minimum(rng.zipf(1.3, size=n), vocab_size) - 1
        files.append((f"f{i:03d}", [vocab[r] for r in ranks]))
        remaining -= n
    return files


def acceptance_corpus(rng):
    """Same distribution as pkg/tests/test_acceptance.py:54-72."""
    num_files = int(rng.integers(1, 65))
    vocab_size = int(rng.integers(1, 5001))
    vocab = [f"w{i}" for i in range(vocab_size)]
    bucket = rng.random()
    if bucket < 0.80:
        total = int(rng.integers(0, 3000))
    elif bucket < 0.95:
        total = int(rng.integers(3000, 20000))
    else:
        total = int(rng.integers(20000, 100001))
    cuts = np.sort(rng.integers(0, total + 1, size=num_files - 1))
    bounds = [0, *cuts.tolist(), total]
    ranks = np.minimum(rng.zipf(1.3, size=total), vocab_size) - 1
    return [(f"f{i:03d}", [vocab[r] for r in ranks[bounds[i]:bounds[i + 1]]])
            for i in range(num_files)]


def c1_files(seed=0):
    """C1: ~1 MB, 10 files, vocab 10k, Zipf s=1.1 clipped (BASELINE configs[0])."""
    rng = np.random.default_rng(seed)
    vocab = [f"w{i}" for i in range(10_000)]
    files = []
    for i in range(10):
        ranks = np.minimum(rng.zipf(1.1, size=20_800), 10_000) - 1
        files.append((f"f{i:02d}", [vocab[r] for r in ranks]))
    return files


G1 = [("A.txt", "a b a b c".split()), ("B.txt", "a b c".split())]


def sequitur_fixtures() -> dict:
    """Fixture name -> token files, for every golden grammar that
    tools/make_golden.py produced with the reference's Sequitur."""
    spill = [f"w{i}" for i in range(70_000)]
    fx = {
        "g1": G1,
        "empty_files": [("a", []), ("b", [])],
        "single_file": [("f", ["x", "x"])],
        "all_equal_counts": [("f", ["u", "v", "w"])],
        "empty_corpus": [("f", [])],
        "word_unique_to_one_file": [("a", ["x"]), ("b", ["x", "zed"])],
        "identical_files": [("a", ["p", "q"]), ("b", ["p", "q"])],
        "many_files_70": [(f"f{i:03d}", [f"w{i % 7}", "common"]) for i in range(70)],
        "spill_70k_l4": [("big", spill + spill[:200])],
    }
    for i in range(16):
        rng = np.random.default_rng(90_000 + i)
        fx[f"fuzz_{i:02d}"] = corpus_tokens(rng, max_files=6, max_tokens=1500, max_vocab=50)
    for i in range(0, 200, 10):
        fx[f"accept_{i:03d}"] = acceptance_corpus(np.random.default_rng(1_000_000 + i))
    fx["c1"] = c1_files()
    return fx
