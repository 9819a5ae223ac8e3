"""B200-native analytics directly on grammar-compressed corpora (G-TADOC).

Drop-in for the reference package's task entry points (`gtadoc.tasks`):
word_count, sort_by_frequency, inverted_index, term_vector, sequence_count,
ranked_inverted_index, run_task and render, backed by hand-written sm_100a
kernels in libgtadoc_b200.so (see include/gtadoc_b200.h).
"""

from .device import DeviceDag, build_dag
from .errors import (CorruptionError, DivergenceError, FormatError, GtadocError,
                     IngestError, ResourceError, UsageError)
from .tasks import (TASK_NAMES, InvertedIndex, RankedInvertedIndex, SequenceCounts,
                    SortedWords, TermVectors, TraversalConfig, WordCounts, first_divergence,
                    inverted_index, output_digest, ranked_inverted_index, render, render_native,
                    run_compact, run_compact_many, run_task, run_tasks, sequence_count, sort_by_frequency, term_vector,
                    word_count)

__version__ = "0.1.0"

__all__ = [
    "DeviceDag", "build_dag", "TraversalConfig", "run_task", "run_compact", "render",
    "first_divergence", "word_count", "sort_by_frequency", "inverted_index", "term_vector",
    "sequence_count", "ranked_inverted_index", "WordCounts", "SortedWords", "InvertedIndex",
    "TermVectors", "SequenceCounts", "RankedInvertedIndex", "TASK_NAMES", "GtadocError",
    "UsageError", "IngestError", "ResourceError", "FormatError", "CorruptionError",
    "DivergenceError", "output_digest", "render_native", "run_compact_many", "run_tasks",
]
