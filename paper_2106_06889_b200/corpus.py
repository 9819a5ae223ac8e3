"""Deterministic synthetic grammar composer (input producer for the configs).

The reference builds its inputs with Sequitur (`src/sequitur.py:251-258`),
which runs at ~10^5 symbols/s in Python, so GB-equivalent corpora cannot be
produced with it.  This module composes a *valid reference grammar* directly
(vectorised numpy, seeded): a stack of rule levels where every body mixes
Zipf-distributed words with Zipf-popular references into the levels below
(heavy multi-parent sharing), and a root whose splitter-delimited segments
(files) reference the upper levels plus fresh words.

Validity is exactly what `build_dag` (`src/dag.py:131-230`) and
`deserialize_grammar` (`src/grammar.py:193-228`) check: symbols in range,
acyclic (children always sit on a lower level), every rule reachable from the
root, splitters only in the root, in order, one after every file.  Rule ids
are randomly permuted so the on-disk order carries no level information.
`tools/make_golden.py` runs the reference on small composed grammars to show
it accepts them and to pin their outputs.

The output is the reference's GTDC byte format (`src/grammar.py:164-174`).
"""

from __future__ import annotations

import math
import struct
from dataclasses import asdict, dataclass

import numpy as np

MAGIC = b"GTDC"
VERSION = 1


@dataclass
class ComposeSpec:
    seed: int = 0
    files: int = 16
    vocab: int = 50_000
    words_target: int = 1_000_000  # W = uncompressed-equivalent words
    levels: int = 12  # rule levels below the root (DAG depth = levels)
    level_rules: int = 10_000  # rules per level
    body_min: int = 2
    body_max: int = 6
    ref_prob: float = 0.15  # P(non-first body slot is a rule reference)
    near_prob: float = 0.75  # P(reference targets the level directly below)
    zipf_words: float = 1.1
    zipf_rules: float = 1.2
    root_levels: int = 3  # the root references the top `root_levels` levels
    fresh_word_prob: float = 0.05  # P(root symbol is a plain word)
    file_size_sigma: float = 0.3  # lognormal spread of file sizes


def _zipf_index(rng: np.random.Generator, s: float, n: int, size: int) -> np.ndarray:
    """Ranks in [0, n) with Zipf(s) popularity, clipped like the reference's
    fuzz corpora (`pkg/tests/conftest.py:45`)."""
    if n <= 0 or size == 0:
        return np.zeros(size, dtype=np.int64)
    return np.minimum(rng.zipf(s, size=size), n).astype(np.int64) - 1


def _coprime_multiplier(n: int) -> int:
    a = 2_654_435_761 % max(n, 1) or 1
    while math.gcd(a, n) != 1:
        a += 1
    return a


def _popular(rank: np.ndarray, level: np.ndarray | int, n: int, salt: int) -> np.ndarray:
    """Bijective rank -> rule-index map per level (which rules are popular)."""
    a = _coprime_multiplier(n)
    off = (np.asarray(level, dtype=np.int64) * 7919 + salt * 104_729) % n
    return (rank * a + off) % n


def serialize_parts(words: list[str], num_splitters: int, lens: np.ndarray,
                    flat: np.ndarray) -> bytes:
    """GTDC bytes (`src/grammar.py:164-174`): header, dictionary (u32 length +
    UTF-8 per word), then per rule u32 body length + u32 symbols, root first."""
    parts = [MAGIC, struct.pack("<BIII", VERSION, len(words), num_splitters, len(lens))]
    for w in words:
        e = w.encode("utf-8")
        parts.append(struct.pack("<I", len(e)))
        parts.append(e)
    lens = np.asarray(lens, dtype=np.int64)
    R = len(lens)
    out = np.empty(R + int(lens.sum()), dtype="<u4")
    starts = np.zeros(R, dtype=np.int64)
    if R > 1:
        starts[1:] = np.cumsum(lens[:-1] + 1)
    out[starts] = lens
    owner = np.repeat(np.arange(R, dtype=np.int64), lens)
    body_start = np.zeros(R, dtype=np.int64)
    if R > 1:
        body_start[1:] = np.cumsum(lens[:-1])
    j = np.arange(len(flat), dtype=np.int64) - body_start[owner]
    out[starts[owner] + 1 + j] = np.asarray(flat, dtype=np.int64)
    parts.append(out.tobytes())
    return b"".join(parts)


def serialize_bodies(words: list[str], num_splitters: int, bodies: list) -> bytes:
    lens = np.asarray([len(b) for b in bodies], dtype=np.int64)
    flat = (np.concatenate([np.asarray(b, dtype=np.int64) for b in bodies])
            if len(bodies) and lens.sum() else np.zeros(0, dtype=np.int64))
    return serialize_parts(words, num_splitters, lens, flat)


def compose(spec: ComposeSpec) -> tuple[bytes, dict]:
    """Compose a grammar; returns (GTDC bytes, stats dict).

    Level k >= 1: every body carries one *cover* reference (a random
    permutation of level k-1, so every rule has a parent) plus, per other
    slot, a Zipf-popular reference with probability `ref_prob` (the heavy
    multi-parent sharing) or a Zipf word.  The root covers the top level the
    same way and adds Zipf-popular references into the top `root_levels`
    levels and fresh words until the word target is reached.
    """
    rng = np.random.default_rng(spec.seed)
    V, F, D, N = spec.vocab, spec.files, spec.levels, spec.level_rules
    rule_base = V + F
    R = 1 + D * N  # ordinal of rule i on level k is 1 + k*N + i
    owners, syms, refs = [], [], []
    exp_len = np.zeros(R, dtype=np.int64)
    for k in range(D):
        lo = 1 + k * N
        m = rng.integers(spec.body_min, spec.body_max + 1, size=N)
        tot = int(m.sum())
        starts = np.concatenate([[0], np.cumsum(m)[:-1]])
        owner = np.repeat(np.arange(lo, lo + N, dtype=np.int64), m)
        sym = np.empty(tot, dtype=np.int64)
        if k == 0:
            is_ref = np.zeros(tot, dtype=bool)
        else:
            cover = starts + (rng.random(N) * m).astype(np.int64)
            is_ref = rng.random(tot) < spec.ref_prob
            is_ref[cover] = False
            nref = int(is_ref.sum())
            near = rng.random(nref) < spec.near_prob
            lvl = np.where(near, k - 1, rng.integers(0, k, size=nref))
            rank = _zipf_index(rng, spec.zipf_rules, N, nref)
            sym[is_ref] = 1 + lvl * N + _popular(rank, lvl, N, spec.seed)
            sym[cover] = 1 + (k - 1) * N + rng.permutation(N)
            is_ref[cover] = True
        sym[~is_ref] = _zipf_index(rng, spec.zipf_words, V, int((~is_ref).sum()))
        contrib = np.where(is_ref, exp_len[np.where(is_ref, sym, 0)], 1)
        np.add.at(exp_len, owner, contrib)
        owners.append(owner)
        syms.append(sym)
        refs.append(is_ref)

    # root: cover the top level, then popular top-level refs + fresh words
    if D:
        cover = 1 + (D - 1) * N + rng.permutation(N)
        cand = np.arange(1 + max(0, D - spec.root_levels) * N, R, dtype=np.int64)
        cover_w = int(exp_len[cover].sum())
        mean_len = float(exp_len[cand].mean())
        mean_sym = spec.fresh_word_prob + (1 - spec.fresh_word_prob) * mean_len
        n_extra = max(0, int((spec.words_target - cover_w) / max(mean_sym, 1.0)))
        is_word = rng.random(n_extra) < spec.fresh_word_prob
        extra = np.empty(n_extra, dtype=np.int64)
        nr = int((~is_word).sum())
        rank = _zipf_index(rng, spec.zipf_rules, len(cand), nr)
        extra[~is_word] = cand[_popular(rank, 0, len(cand), spec.seed + 1)]
        extra[is_word] = _zipf_index(rng, spec.zipf_words, V, int(is_word.sum()))
        rsym = np.concatenate([cover, extra])
        risr = np.concatenate([np.ones(N, dtype=bool), ~is_word])
    else:
        rsym = _zipf_index(rng, spec.zipf_words, V, spec.words_target)
        risr = np.zeros(len(rsym), dtype=bool)
    order = rng.permutation(len(rsym))
    rsym, risr = rsym[order], risr[order]
    rlen = np.where(risr, exp_len[np.where(risr, rsym, 0)], 1)
    sizes = rng.lognormal(0.0, spec.file_size_sigma, size=F)
    frac = np.cumsum(sizes) / sizes.sum()
    csum = np.cumsum(rlen)
    total = int(csum[-1]) if len(csum) else 0
    cut = np.searchsorted(csum, frac * total, side="left") + 1
    cut = np.maximum.accumulate(np.minimum(cut, len(rsym)))
    cut[-1] = len(rsym)
    seg_lo = np.concatenate([[0], cut[:-1]])

    # final rule ids: random permutation of the non-root ordinals
    perm = np.zeros(R, dtype=np.int64)
    perm[1:] = rng.permutation(np.arange(1, R, dtype=np.int64))

    def enc(sym, isref):
        return np.where(isref, rule_base + perm[np.where(isref, sym, 0)], sym)

    root_parts = []
    for f in range(F):
        s = slice(seg_lo[f], cut[f])
        root_parts.append(enc(rsym[s], risr[s]))
        root_parts.append(np.asarray([V + f], dtype=np.int64))
    root_body = np.concatenate(root_parts) if root_parts else np.zeros(0, np.int64)
    owner_all = np.concatenate([np.zeros(len(root_body), np.int64)] + [perm[o] for o in owners])
    sym_all = np.concatenate([root_body] + [enc(s, r) for s, r in zip(syms, refs)])
    order = np.argsort(owner_all, kind="stable")
    lens = np.bincount(owner_all, minlength=R).astype(np.int64)
    blob = serialize_parts([f"w{i}" for i in range(V)], F, lens, sym_all[order])
    E = int(lens.sum())
    stats = dict(spec=asdict(spec), R=int(R), E=E, L0=int(lens[0]), W=total, F=F, V=V,
                 depth=D, rho=total / max(1, E), bytes=len(blob))
    return blob, stats


# -- named configurations --------------------------------

def config_spec(name: str, seed: int | None = None, scale: float = 1.0) -> ComposeSpec:
    """Composer settings for the BASELINE.json configs.  `scale` shrinks the
    word target and rule counts together for parity-sized variants."""
    def sd(default):
        return default if seed is None else seed
    if name == "c2":  # 1 GB-equivalent, few large files, deep DAG, heavy sharing
        return ComposeSpec(seed=sd(2), files=16, vocab=100_000,
                           words_target=int(170_000_000 * scale), levels=24,
                           level_rules=max(64, int(35_000 * scale)), ref_prob=0.115,
                           root_levels=4, fresh_word_prob=0.1)
    if name == "c3":  # 4 GB-equivalent, 100k small files over a shared pool
        return ComposeSpec(seed=sd(3), files=max(4, int(100_000 * scale)), vocab=50_000,
                           words_target=int(700_000_000 * scale), levels=6,
                           level_rules=max(64, int(8_000 * scale)), ref_prob=0.35,
                           root_levels=2, fresh_word_prob=0.15, file_size_sigma=0.5)
    if name == "c4":  # 10 GB-equivalent, 3-gram sequence count
        return ComposeSpec(seed=sd(4), files=64, vocab=100_000,
                           words_target=int(1_700_000_000 * scale), levels=28,
                           level_rules=max(64, int(400_000 * scale)), ref_prob=0.12,
                           root_levels=4, fresh_word_prob=0.1)
    if name == "c5":  # 50 GB-equivalent, vocab 1M
        return ComposeSpec(seed=sd(5), files=64, vocab=1_000_000,
                           words_target=int(8_000_000_000 * scale), levels=30,
                           level_rules=max(64, int(600_000 * scale)), ref_prob=0.12,
                           root_levels=4, fresh_word_prob=0.1)
    raise ValueError(f"unknown config {name!r}")
