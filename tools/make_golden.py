#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Run in the build container only (the reference lives at /root/reference and
does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc \
        python tools/make_golden.py

For every fixture it stores the GTDC bytes (gzip) and, from the reference's
own engine (`gtadoc.tasks.run_task`, numba backend, both strategies, which
must agree), the sha256 + line count of `render(...)` for all six tasks and
several sequence lengths, plus digests of the `build_dag` arrays and the
reference's per-round frontiers (the level schedule).  Small fixtures are
also cross-checked against the decompress-then-count oracle
(`gtadoc.tasks.oracle_task`).  Error fixtures store the exception class and
message the reference raises.

Fixture sources: the reference test suite's own inputs (G1
`pkg/tests/conftest.py:12-28`, `manual_grammar` shapes from
`pkg/tests/test_dag.py`, `test_engine.py`, `test_sequence.py`, the task edge
cases of `test_tasks.py`, the spill corpus `test_sequence.py:194-216`), the
fuzz generators (`conftest.py:31-48`, `test_acceptance.py:54-72`), the C1
config, and small grammars from our composer (to prove the reference accepts
composer output).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REPO = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(REPO))

from gtadoc import oracle  # noqa: E402  (reference package)
from gtadoc.dag import build_dag  # noqa: E402
from gtadoc.engine import (TraversalConfig, TraversalState,  # noqa: E402
                           init_bottom_up_masks, init_top_down_masks)
from gtadoc.errors import GtadocError  # noqa: E402
from gtadoc.grammar import Grammar, deserialize_grammar, serialize_grammar  # noqa: E402
from gtadoc.ingest import Dictionary, build_corpus_stream  # noqa: E402
from gtadoc.sequitur import infer_grammar  # noqa: E402
from gtadoc.tasks import oracle_task, render, run_task  # noqa: E402

from paper_2106_06889_b200.corpus import ComposeSpec, compose, config_spec  # noqa: E402

OUT = REPO / "tests" / "golden"
GRAM = OUT / "grammars"

WORD_TASKS = ["wordcount", "sort", "invertedindex", "termvector"]
SEQ_TASKS = ["seqcount", "rankedinvertedindex"]


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def arr_sha(a) -> str:
    return sha(np.ascontiguousarray(np.asarray(a, dtype="<i8")).tobytes())


def manual(num_words, bodies, num_splitters=0):
    d = Dictionary(words=[f"w{i}" for i in range(num_words)], num_splitters=num_splitters)
    return Grammar(dictionary=d, bodies=[np.asarray(b, dtype=np.int64) for b in bodies])


def sequitur(files):
    d, s = build_corpus_stream(files)
    return infer_grammar(d, s)


sys.path.insert(0, str(REPO / "tests"))
from corpora import acceptance_corpus, c1_files, corpus_tokens  # noqa: E402,F401  (shared generators)


def td_rounds(dag):
    """Per-rule round index of the reference's top-down traversal
    (`src/engine.py:196-227`): replays its mask protocol."""
    from gtadoc.engine import Runner, partition_work
    state = TraversalState(dag)
    init_top_down_masks(dag, state)
    cfg = TraversalConfig(backend="numba")
    runner = Runner(cfg)
    rnd = np.zeros(dag.num_rules, dtype=np.int64)
    changes = np.zeros(1, dtype=np.int64)
    sub_counts = np.diff(dag.sub_off)
    k = 0
    while True:
        frontier = np.flatnonzero(state.mask)
        if frontier.size == 0:
            break
        k += 1
        rnd[frontier] = k
        lengths = sub_counts[frontier]
        units = partition_work(frontier, lengths, int(lengths.sum()), cfg)
        runner.run("topdown_round",
                   (dag.sub_ids, dag.sub_freqs, dag.sub_off, state.wmat, state.nfiles,
                    state.cur_in, dag.num_in_edge, state.mask, changes, *units),
                   len(units[0]))
        state.mask[frontier] = 0
    runner.close()
    return rnd, state.weight


def bu_rounds(dag):
    """Per-rule round index of the reference's bottom-up readiness protocol
    (`src/engine.py:313-335`)."""
    state = TraversalState(dag)
    init_bottom_up_masks(dag, state)
    rnd = np.zeros(dag.num_rules, dtype=np.int64)
    k = 0
    while True:
        ready = np.flatnonzero(state.mask)
        if ready.size == 0:
            break
        k += 1
        rnd[ready] = k
        for r in ready:
            for j in range(dag.par_off[r], dag.par_off[r + 1]):
                p = int(dag.par_ids[j])
                state.cur_out[p] += int(dag.par_freqs[j])
                if p != 0 and state.cur_out[p] == dag.num_out_edge[p]:
                    state.mask[p] = 1
        state.mask[ready] = 0
    return rnd


def dag_record(dag):
    rec = dict(
        num_rules=dag.num_rules, num_files=dag.num_files, depth=int(dag.depth),
        total_elements=int(dag.total_elements),
        segments=[list(map(int, s)) for s in dag.segments] if dag.num_files <= 200 else None,
        segments_sha=arr_sha(np.asarray(dag.segments, dtype=np.int64).reshape(-1)),
        W=int(dag.exp_len[0]),
    )
    for name in ["own_ids", "own_freqs", "own_off", "own_token_count", "sub_ids",
                 "sub_freqs", "sub_off", "par_ids", "par_freqs", "par_off",
                 "num_in_edge", "num_out_edge", "root_freq", "exp_len"]:
        rec[name] = arr_sha(getattr(dag, name))
    rec["segment_token_counts"] = arr_sha(dag.segment_token_counts)
    td, weight = td_rounds(dag)
    rec["td_round"] = arr_sha(td)
    rec["td_rounds"] = int(td.max()) if len(td) else 0
    rec["weight"] = arr_sha(weight)
    bu = bu_rounds(dag)
    rec["bu_round"] = arr_sha(bu)
    rec["bu_rounds"] = int(bu.max()) if len(bu) else 0
    if dag.num_rules <= 64:
        rec["weight_list"] = [int(x) for x in weight]
        rec["td_round_list"] = [int(x) for x in td]
        rec["bu_round_list"] = [int(x) for x in bu]
    return rec


def outputs(g, dag, seq_lens, seq=True, check_oracle=False, strategies=("topdown", "bottomup")):
    res = {}
    files = oracle.decompress_files(g) if check_oracle else None
    jobs = [(t, 3) for t in WORD_TASKS]
    if seq:
        jobs += [(t, l) for t in SEQ_TASKS for l in seq_lens]
    for task, l in jobs:
        texts = set()
        for strat in strategies:
            cfg = TraversalConfig(strategy=strat, backend="numba")
            texts.add(render(run_task(dag, task, cfg, l), g.dictionary))
        assert len(texts) == 1, (task, l, "strategies disagree")
        text = texts.pop()
        if check_oracle:
            exp = render(oracle_task(g, task, l, files), g.dictionary)
            assert exp == text, (task, l, "oracle disagrees")
        key = task if task in WORD_TASKS else f"{task}@{l}"
        ent = dict(sha256=sha(text.encode()), lines=text.count("\n"), bytes=len(text.encode()))
        if len(text) <= 4096:
            ent["text"] = text
        res[key] = ent
    return res


def main():
    GRAM.mkdir(parents=True, exist_ok=True)
    expected = {}
    t_all = time.time()

    def add(name, g=None, blob=None, seq_lens=(1, 2, 3, 4), seq=True, check_oracle=True,
            kind="engine", strategies=("topdown", "bottomup")):
        t0 = time.time()
        if blob is None:
            blob = serialize_grammar(g)
        (GRAM / f"{name}.gtdc.gz").write_bytes(gzip.compress(blob, 9, mtime=0))
        try:
            gg = deserialize_grammar(blob)
            dag = build_dag(gg)
        except GtadocError as exc:
            expected[name] = dict(kind="error", error=type(exc).__name__, message=str(exc),
                                  exit_code=exc.exit_code)
            print(f"{name:28s} error {type(exc).__name__}: {exc}")
            return
        rec = dict(kind=kind, gtdc_sha256=sha(blob), dag=dag_record(dag))
        rec["outputs"] = outputs(gg, dag, seq_lens, seq=seq, check_oracle=check_oracle,
                                 strategies=strategies)
        rec["seq_lens"] = list(seq_lens) if seq else []
        expected[name] = rec
        print(f"{name:28s} R={dag.num_rules:7d} E={dag.total_elements:8d} F={dag.num_files:6d} "
              f"W={int(dag.exp_len[0]):12d} d={dag.depth:3d}  {time.time() - t0:6.1f}s", flush=True)

    # -- reference fixtures --------------------------------------------------
    G1 = [("A.txt", "a b a b c".split()), ("B.txt", "a b c".split())]
    add("g1", sequitur(G1), seq_lens=(1, 2, 3, 4, 9, 40))
    add("empty_files", sequitur([("a", []), ("b", [])]))
    add("single_file", sequitur([("f", ["x", "x"])]))
    add("all_equal_counts", sequitur([("f", ["u", "v", "w"])]))
    add("empty_corpus", sequitur([("f", [])]))
    add("word_unique_to_one_file", sequitur([("a", ["x"]), ("b", ["x", "zed"])]))
    add("identical_files", sequitur([("a", ["p", "q"]), ("b", ["p", "q"])]))
    add("many_files_70", sequitur([(f"f{i:03d}", [f"w{i % 7}", "common"]) for i in range(70)]))
    add("root_only", manual(2, [[0, 1, 0]]))
    add("chain", manual(1, [[2], [3, 3], [0]]))
    add("all_leaf", manual(1, [[2, 2], [0]]))
    add("two_leaves", manual(2, [[3, 4, 3, 4], [0], [1]]))
    add("scaled_merge", manual(1, [[2, 2], [3, 3], [0]]))
    add("bounds_leaf", manual(1, [[2, 2], [0, 0, 0]]))
    add("middle_child_owned", manual(5, [[0, 6, 4, 0, 6, 4], [1, 2, 3]]))
    add("long_child_head_gap_tail", manual(10, [[11, 11], list(range(10))]))
    add("root_only_segment", manual(1, [[0, 1]], num_splitters=1))
    add("duplicate_words", manual(2, [[0, 0, 1, 0]]))
    add("empty_rule_body", manual(2, [[0, 4, 1, 4, 2], []], num_splitters=1))
    add("splitter_inside_rule", manual(2, [[5, 2, 0, 5, 3], [0, 2, 1]], num_splitters=2),
        check_oracle=False)
    # deep doubling chain: counts 2^40, the decompressing oracle cannot run it;
    # per-file gram tables are sized by tokens in the reference, so no seq tasks
    depth = 40
    add("doubling_chain_40", manual(1, [[2]] + [[3 + i, 3 + i] for i in range(depth - 1)] + [[0]]),
        seq=False, check_oracle=False)
    spill = [f"w{i}" for i in range(70_000)]
    add("spill_70k_l4", sequitur([("big", spill + spill[:200])]), seq_lens=(4,), check_oracle=True)

    # -- fuzz (reference generators) ------------------------------------------
    for i in range(16):
        rng = np.random.default_rng(90_000 + i)
        add(f"fuzz_{i:02d}", sequitur(corpus_tokens(rng, max_files=6, max_tokens=1500,
                                                    max_vocab=50)), seq_lens=(2, 3, 4))
    for i in range(0, 200, 10):
        rng = np.random.default_rng(1_000_000 + i)
        add(f"accept_{i:03d}", sequitur(acceptance_corpus(rng)), seq_lens=(3,))

    # -- composer output accepted by the reference -----------------------------
    for seed in range(6):
        spec = ComposeSpec(seed=seed, files=1 + seed * 3, vocab=40 + 30 * seed,
                           words_target=4000 + 3000 * seed, levels=4 + seed,
                           level_rules=30 + 10 * seed, ref_prob=0.2, root_levels=2)
        blob, _ = compose(spec)
        add(f"composed_{seed}", blob=blob, seq_lens=(2, 3), kind="composed")
    blob, _ = compose(config_spec("c2", scale=0.0002))
    add("composed_c2_tiny", blob=blob, seq_lens=(3,), kind="composed", check_oracle=True)
    blob, _ = compose(config_spec("c3", scale=0.0005))
    add("composed_c3_tiny", blob=blob, seq_lens=(3,), kind="composed", check_oracle=True)

    # -- C1 (BASELINE configs[0]) ---------------------------------------------
    add("c1", sequitur(c1_files()), seq_lens=(3,), check_oracle=True)

    # -- errors --------------------------------------------------------------
    g1b = serialize_grammar(sequitur(G1))
    add("err_bad_magic", blob=b"GTDX" + g1b[4:])
    add("err_short", blob=b"GT")
    add("err_truncated", blob=g1b[:-3])
    add("err_trailing", blob=g1b + b"\x00")
    add("err_version", blob=g1b[:4] + b"\x02" + g1b[5:])
    import struct
    add("err_zero_rules", blob=b"GTDC" + struct.pack("<BIII", 1, 0, 0, 0))
    add("err_symbol_range", blob=serialize_grammar(manual(1, [[0, 5]])))
    add("err_bad_utf8", blob=b"GTDC" + struct.pack("<BIII", 1, 1, 0, 1)
        + struct.pack("<I", 1) + b"\xff" + struct.pack("<II", 1, 0))
    add("err_cycle", manual(1, [[2], [3, 3], [2, 0]]))
    add("err_unreachable", manual(1, [[0], [0, 0]]))
    add("err_splitter_order", manual(1, [[0, 2, 0, 1]], num_splitters=2))
    add("err_after_last_splitter", manual(1, [[0, 1, 0]], num_splitters=1))
    add("err_missing_splitters", manual(1, [[0, 1]], num_splitters=2))
    add("err_self_reference", manual(1, [[1]]))

    meta = dict(generated_by="tools/make_golden.py", reference="/root/reference/pkg (gtadoc 0.1.0)",
                backend="numba", seconds=round(time.time() - t_all, 1))
    (OUT / "expected.json").write_text(json.dumps(dict(meta=meta, fixtures=expected), indent=1,
                                                  sort_keys=True))
    print(f"done in {time.time() - t_all:.1f}s, {len(expected)} fixtures")


if __name__ == "__main__":
    main()
