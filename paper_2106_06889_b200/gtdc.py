"""Host-side GTDC helpers: the dictionary (for `render`) and file loading.

The byte format is the reference's (`src/grammar.py:1-15,164-228`).  Rule
bodies are parsed, validated and flattened by the C-ABI (`gt_open`); Python
only needs the word strings to render TSV, so the dictionary is decoded
lazily.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass, field

from .errors import FormatError


@dataclass
class Dictionary:
    """ingest.py:46-84 (words + splitter block; lookup helpers)."""

    words: list[str]
    num_splitters: int
    _index: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def num_words(self) -> int:
        return len(self.words)

    @property
    def num_terminals(self) -> int:
        return len(self.words) + self.num_splitters

    def word_id(self, word: str) -> int:
        if not self._index:
            self._index = {w: i for i, w in enumerate(self.words)}
        return self._index[word]

    def is_word(self, sym: int) -> bool:
        return 0 <= sym < self.num_words

    def is_splitter(self, sym: int) -> bool:
        return self.num_words <= sym < self.num_terminals


def read_dictionary(blob: bytes) -> Dictionary:
    """Decode the dictionary section (grammar.py:193-215).  Assumes the blob
    already passed gt_open's validation."""
    if len(blob) < 17 or blob[:4] != b"GTDC":
        raise FormatError("bad magic: not a GTDC file")
    _, nw, ns, _ = struct.unpack_from("<BIII", blob, 4)
    pos = 17
    words = []
    mv = memoryview(blob)
    for _ in range(nw):
        (n,) = struct.unpack_from("<I", blob, pos)
        pos += 4
        words.append(str(mv[pos:pos + n], "utf-8"))
        pos += n
    return Dictionary(words=words, num_splitters=ns)


@dataclass
class GrammarView:
    """Just enough of the reference `Grammar` for `render(out, g.dictionary)`."""

    blob: bytes
    _dictionary: Dictionary | None = None

    @property
    def dictionary(self) -> Dictionary:
        if self._dictionary is None:
            self._dictionary = read_dictionary(self.blob)
        return self._dictionary
