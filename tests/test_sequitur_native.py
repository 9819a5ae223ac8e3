"""Native compressor (csrc/sequitur.cpp) == the reference's Sequitur output,
byte for byte: every golden grammar that tools/make_golden.py produced by
running the reference's ingest + infer_grammar + serialize_grammar is
regenerated from the same deterministic corpus (tests/corpora.py) and
compressed natively (host code, no GPU)."""

from __future__ import annotations

import pytest

from conftest import expected, gtdc
from corpora import sequitur_fixtures

FIX = sequitur_fixtures()


def as_bytes(files):
    return [(name, " ".join(toks).encode()) for name, toks in files]


@pytest.mark.parametrize("name", sorted(FIX))
def test_native_compressor_reproduces_reference_grammar(name):
    from paper_2106_06889_b200.compress import compress_files
    blob, stats = compress_files(as_bytes(FIX[name]))
    assert blob == gtdc(name)
    assert stats["files"] == len(FIX[name])


def test_whitespace_and_utf8_rules():
    from paper_2106_06889_b200 import IngestError
    from paper_2106_06889_b200.compress import compress_files
    # Python str.split() separators, including Unicode spaces
    raw = "a\tb c d\n\x1ce　f  g".encode()
    blob, stats = compress_files([("x", raw)])
    assert stats["vocabulary"] == 7
    with pytest.raises(IngestError, match=r"^b\.txt: invalid UTF-8 at byte offset 4$"):
        compress_files([("a.txt", b"ok"), ("b.txt", b"bad \xff\xfe here")])
    with pytest.raises(IngestError, match="byte offset 2"):
        compress_files([("c", b"ab\xe2\x82")])  # truncated 3-byte sequence


def test_compress_dir_order_and_usage(tmp_path):
    from paper_2106_06889_b200 import UsageError
    from paper_2106_06889_b200.compress import compress_dir
    (tmp_path / "B.txt").write_text("a b c")
    (tmp_path / "A.txt").write_text("a b a b c")
    blob, _ = compress_dir(tmp_path)
    assert blob == gtdc("g1")  # lexicographic order: A.txt, B.txt
    empty = tmp_path / "empty"
    empty.mkdir()
    with pytest.raises(UsageError, match="no regular files"):
        compress_dir(empty)
