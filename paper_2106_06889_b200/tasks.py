"""The six analytics tasks — drop-in mirror of the reference's `src/tasks.py`.

Same names, signatures, output containers and rendering as
`tasks.py:122-263`; the work runs in libgtadoc_b200.so (sm_100a kernels)
through the C-ABI in include/gtadoc_b200.h.  `dag` is a `DeviceDag` (the
device-resident counterpart of the reference's `Dag`, built by `build_dag`
from a `.gtdc` blob) and `cfg` a `TraversalConfig` with the reference's
fields (engine.py:34-48).  There is no CPU fallback: without the CUDA
library every call raises.

Ordering rules (tasks.py:1-21) are enforced by the device assembly kernels,
so `render` only formats.
"""

from __future__ import annotations

from dataclasses import dataclass

from ._abi import STRATEGY_IDS, TASK_IDS, TASK_NAMES, Compact, to_container
from .errors import UsageError

DEFAULT_SEQ_LEN = 3
STRATEGIES = ("auto", "topdown", "bottomup")


@dataclass
class TraversalConfig:
    """engine.py:34-48.  `workers` is the number of GPUs (file-range shards)
    a task runs on: workers > 1 shards the corpus with shard.ShardedDag (the
    DAG built once and replicated by peer copies, results combined on the
    first device)."""

    strategy: str = "auto"
    workers: int = 1
    chunk_factor: int = 16
    file_set_width: int = 64
    backend: str | None = None

    def __post_init__(self) -> None:
        if self.strategy not in STRATEGIES:
            raise UsageError(f"unknown strategy {self.strategy!r}")
        if self.workers < 1:
            raise UsageError("workers must be >= 1")
        if self.chunk_factor < 1:
            raise UsageError("chunk factor must be >= 1")


@dataclass
class WordCounts:
    counts: dict[int, int]


@dataclass
class SortedWords:
    pairs: list[tuple[int, int]]


@dataclass
class InvertedIndex:
    files_of: dict[int, list[int]]


@dataclass
class TermVectors:
    vectors: list[list[tuple[int, int]]]


@dataclass
class SequenceCounts:
    per_file: list[dict[tuple[int, ...], int]]


@dataclass
class RankedInvertedIndex:
    ranked: dict[tuple[int, ...], list[tuple[int, int]]]


def run_compact(dag, task: str, cfg: TraversalConfig | None = None,
                seq_len: int = DEFAULT_SEQ_LEN) -> Compact:
    """run_task returning compact render-ordered arrays (no Python dicts)."""
    if task not in TASK_IDS:
        raise UsageError(f"unknown task {task!r}; expected one of {', '.join(TASK_NAMES)}")
    cfg = cfg or TraversalConfig()
    if task in ("seqcount", "rankedinvertedindex") and seq_len < 1:
        raise UsageError("sequence length must be >= 1")
    return _workers(dag, cfg).run(TASK_IDS[task], seq_len, STRATEGY_IDS[cfg.strategy], cfg.file_set_width)


def _workers(dag, cfg: TraversalConfig):
    """The handle a task runs on: a reference `Dag` / `Grammar` is loaded
    onto the device once (device.as_device_dag), and with cfg.workers > 1 a
    DeviceDag is sharded over that many devices (other handles, e.g. the
    test oracle, run as given)."""
    from .device import as_device_dag
    dag = as_device_dag(dag)
    if cfg.workers > 1 and hasattr(dag, "sharded"):
        return dag.sharded(cfg.workers)
    return dag


def run_compact_many(dag, tasks, cfg: TraversalConfig | None = None,
                     seq_len: int = DEFAULT_SEQ_LEN) -> list[Compact]:
    """Several tasks in one call, one Compact per task (same results as
    run_compact each).  On the device, word count / sort together with the
    inverted index share ONE top-down pass (gt_run_many)."""
    cfg = cfg or TraversalConfig()
    for task in tasks:
        if task not in TASK_IDS:
            raise UsageError(f"unknown task {task!r}; expected one of {', '.join(TASK_NAMES)}")
    if any(t in ("seqcount", "rankedinvertedindex") for t in tasks) and seq_len < 1:
        raise UsageError("sequence length must be >= 1")
    dag = _workers(dag, cfg)
    if hasattr(dag, "run_many"):
        return dag.run_many([TASK_IDS[t] for t in tasks], seq_len, STRATEGY_IDS[cfg.strategy],
                            cfg.file_set_width)
    return [run_compact(dag, t, cfg, seq_len) for t in tasks]


def run_tasks(dag, tasks, cfg: TraversalConfig, seq_len: int = DEFAULT_SEQ_LEN) -> list:
    """run_task (tasks.py:171-185) for several tasks at once: the reference's
    output containers, in the order of `tasks`."""
    return [to_container(c) for c in run_compact_many(dag, tasks, cfg, seq_len)]


def output_digest(dag, task: str, cfg: TraversalConfig | None = None,
                  seq_len: int = DEFAULT_SEQ_LEN) -> tuple[str, int]:
    """sha256 hex + byte length of `render(run_task(...))` — the reference
    CLI manifest's outputDigest (cli.py:121-133) — rendered natively
    (render.cpp) without building the Python containers or the text."""
    from .device import as_device_dag
    from .native import NativeDict
    dag = as_device_dag(dag)
    return NativeDict(dag.grammar.blob).digest(run_compact(dag, task, cfg, seq_len))


def render_native(dag, task: str, cfg: TraversalConfig | None = None,
                  seq_len: int = DEFAULT_SEQ_LEN) -> str:
    """`render(run_task(...), dag.grammar.dictionary)`, rendered natively."""
    from .device import as_device_dag
    from .native import NativeDict
    dag = as_device_dag(dag)
    return NativeDict(dag.grammar.blob).render(run_compact(dag, task, cfg, seq_len))


def word_count(dag, cfg: TraversalConfig) -> WordCounts:
    return to_container(run_compact(dag, "wordcount", cfg))


def sort_by_frequency(dag, cfg: TraversalConfig) -> SortedWords:
    return to_container(run_compact(dag, "sort", cfg))


def inverted_index(dag, cfg: TraversalConfig) -> InvertedIndex:
    return to_container(run_compact(dag, "invertedindex", cfg))


def term_vector(dag, cfg: TraversalConfig) -> TermVectors:
    return to_container(run_compact(dag, "termvector", cfg))


def sequence_count(dag, cfg: TraversalConfig, seq_len: int = DEFAULT_SEQ_LEN) -> SequenceCounts:
    return to_container(run_compact(dag, "seqcount", cfg, seq_len))


def ranked_inverted_index(dag, cfg: TraversalConfig,
                          seq_len: int = DEFAULT_SEQ_LEN) -> RankedInvertedIndex:
    return to_container(run_compact(dag, "rankedinvertedindex", cfg, seq_len))


def run_task(dag, task: str, cfg: TraversalConfig, seq_len: int = DEFAULT_SEQ_LEN):
    """tasks.py:171-185"""
    if task not in TASK_IDS:
        raise UsageError(f"unknown task {task!r}; expected one of {', '.join(TASK_NAMES)}")
    return to_container(run_compact(dag, task, cfg, seq_len))


# -- rendering (tasks.py:233-263, byte-for-byte) --------------------------------


def render(output, dictionary) -> str:
    words = dictionary.words
    lines: list[str] = []
    if isinstance(output, WordCounts):
        for w in sorted(output.counts):
            lines.append(f"{words[w]}\t{output.counts[w]}")
    elif isinstance(output, SortedWords):
        for w, c in output.pairs:
            lines.append(f"{words[w]}\t{c}")
    elif isinstance(output, InvertedIndex):
        for w in sorted(output.files_of):
            files = "\t".join(str(f) for f in output.files_of[w])
            lines.append(f"{words[w]}\t{files}")
    elif isinstance(output, TermVectors):
        for f, vec in enumerate(output.vectors):
            for w, c in vec:
                lines.append(f"{f}\t{words[w]}\t{c}")
    elif isinstance(output, SequenceCounts):
        for f, table in enumerate(output.per_file):
            ordered = sorted(table.items(), key=lambda kv: (-kv[1], kv[0]))
            for gram, c in ordered:
                text = " ".join(words[w] for w in gram)
                lines.append(f"{f}\t{text}\t{c}")
    elif isinstance(output, RankedInvertedIndex):
        for gram in sorted(output.ranked):
            text = " ".join(words[w] for w in gram)
            pairs = "\t".join(f"{f}:{c}" for f, c in output.ranked[gram])
            lines.append(f"{text}\t{pairs}")
    else:
        raise UsageError(f"cannot render {type(output).__name__}")
    return "".join(line + "\n" for line in lines)


def first_divergence(expected: str, actual: str) -> str | None:
    """tasks.py:266-278"""
    exp_lines = expected.splitlines()
    act_lines = actual.splitlines()
    for i, (e, a) in enumerate(zip(exp_lines, act_lines)):
        if e != a:
            return f"line {i + 1}: expected {e!r}, got {a!r}"
    if len(exp_lines) != len(act_lines):
        longer = "expected" if len(exp_lines) > len(act_lines) else "actual"
        i = min(len(exp_lines), len(act_lines))
        extra = exp_lines[i] if longer == "expected" else act_lines[i]
        return f"line {i + 1}: {longer} side has extra record {extra!r}"
    return None
